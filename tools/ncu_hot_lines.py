#!/usr/bin/env python3
"""Hot source lines of a kernel from `ncu -i rep --page source --csv --print-source sass,cuda`
(optionally gzipped).  usage: ncu_hot_lines.py <csv[.gz]> [kernel substring] [top N]
Only the CUDA-C rows are counted (the SASS rows under them repeat the same counters)."""
import csv
import gzip
import sys


def main():
    path = sys.argv[1]
    want = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    fh = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    fname = func = None
    hdr = None
    agg = {}
    for row in csv.reader(fh):
        if len(row) == 2 and row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if len(row) == 2 and row[0] == "Function Name":
            func = row[1]
            continue
        if row and row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or not row or not row[0] or want not in (func or ""):
            continue
        d = dict(zip(hdr, row))

        def f(k):
            try:
                return float(d.get(k, "0") or 0)
            except ValueError:
                return 0.0

        key = (func.split("(")[0][-40:], fname, row[0])
        a = agg.setdefault(key, [row[1].strip()[:70], 0, 0, 0, 0, 0, 0, 0])
        a[1] += f("# Samples")
        a[2] += f("Instructions Executed")
        a[3] += f("L1 Wavefronts Shared")
        a[4] += f("L1 Tag Requests Global")
        a[5] += f("L2 Theoretical Sectors Global")
        a[6] += f("stall_long_sb")
        a[7] += f("stall_barrier")
    tot = [sum(a[i] for a in agg.values()) or 1 for i in range(1, 8)]
    print("totals: samples %d inst %d shared wavefronts %d global tags %d l2 sectors %d" % tuple(tot[:5]))
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print("%-22s %-12s %5s | samp %4.1f%% inst %4.1f%% shwf %4.1f%% tags %4.1f%% l2s %4.1f%% longsb %4.1f%% bar %4.1f%% | %s" % (
            k[0][-22:], k[1][:12], k[2], 100 * a[1] / tot[0], 100 * a[2] / tot[1], 100 * a[3] / tot[2],
            100 * a[4] / tot[3], 100 * a[5] / tot[4], 100 * a[6] / tot[5], 100 * a[7] / tot[6], a[0]))


if __name__ == "__main__":
    main()
