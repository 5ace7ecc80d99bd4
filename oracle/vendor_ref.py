"""Recipe that places the UNMODIFIED reference package under oracle/_ref/ --
TEST INFRASTRUCTURE ONLY.

    python -m oracle.vendor_ref            # copies /root/reference/pkg/src/ptsbe -> oracle/_ref/ptsbe

The reference is pure Python (13 source files, no build step), so "building"
it is a verbatim copy of its package directory.  oracle/_ref/ is git-ignored
(no reference source enters the history) but not gpurun-ignored, so the copy
travels to the GPU box, where `bench.py --impl reference` and the
`cpu_baseline` leg time the reference's OWN sampler loop on the host cores
(`cpu_baseline.kind = "reference"`).  A SHA-256 manifest of the copied files is
written next to them so a run can state exactly what it timed.
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = "/root/reference/pkg/src/ptsbe"
DST_ROOT = os.path.join(HERE, "_ref")
DST = os.path.join(DST_ROOT, "ptsbe")


def available() -> bool:
    """True when a vendored copy exists (this container after build(), or the GPU box)."""
    return os.path.isfile(os.path.join(DST, "engine.py"))


def vendor(force: bool = False) -> bool:
    """Copy the reference package; returns True when oracle/_ref/ptsbe exists afterwards."""
    if not os.path.isdir(SRC):
        return available()
    if available() and not force:
        return True
    if os.path.isdir(DST):
        shutil.rmtree(DST)
    os.makedirs(DST_ROOT, exist_ok=True)
    shutil.copytree(SRC, DST, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    manifest = {}
    for base, _, files in os.walk(DST):
        for name in sorted(files):
            path = os.path.join(base, name)
            with open(path, "rb") as fp:
                manifest[os.path.relpath(path, DST)] = hashlib.sha256(fp.read()).hexdigest()
    with open(os.path.join(DST_ROOT, "MANIFEST.json"), "w") as fp:
        json.dump({"source": SRC, "files": manifest}, fp, indent=1)
    return True


def load():
    """Import the vendored reference package (module name `ptsbe`)."""
    if not available():
        raise RuntimeError("oracle/_ref/ptsbe is missing: run `python -m oracle.vendor_ref` in the build container")
    sys.dont_write_bytecode = True
    if DST_ROOT not in sys.path:
        sys.path.insert(0, DST_ROOT)
    import ptsbe  # noqa: F401

    return ptsbe


if __name__ == "__main__":
    ok = vendor(force=True)
    print("oracle/_ref/ptsbe:", "present" if ok else "reference sources not found")
