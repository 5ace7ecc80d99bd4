"""bench.py's own launcher: `python bench.py --gpus N` with WORLD_SIZE unset starts N ranks itself
(`--gpus` used to be echoed only), refuses a world size that contradicts `--gpus`,
and the N-rank strong-scaling run reproduces the single-process histogram."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _run(args, env_extra=None, timeout=600):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(env_extra or {})
    proc = subprocess.run([sys.executable, BENCH] + args, capture_output=True, text=True, env=env, timeout=timeout)
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    return proc, (json.loads(lines[-1]) if lines else None)


def test_gpus_flag_spawns_ranks_dry_run():
    one, doc1 = _run(["--gpus", "1", "--dry-run", "--sets", "12", "--shots", "5", "--scaling", "strong"])
    two, doc2 = _run(["--gpus", "2", "--dry-run", "--sets", "12", "--shots", "5", "--scaling", "strong"])
    assert one.returncode == 0 and two.returncode == 0, two.stderr[-2000:]
    assert doc1["n_gpus"] == 1 and doc2["n_gpus"] == 2
    assert doc2["scaling"] == "strong" and doc2["error_sets_total"] == 12 and doc2["shots_total"] == 60
    assert doc1["histogram_checksum"] == doc2["histogram_checksum"]
    _, weak = _run(["--gpus", "2", "--dry-run", "--sets", "12", "--shots", "5"])
    assert weak["n_gpus"] == 2 and weak["error_sets_total"] == 24


def test_world_size_must_match_gpus():
    proc, doc = _run(["--gpus", "4", "--dry-run"], env_extra={"WORLD_SIZE": "2", "RANK": "0"})
    assert proc.returncode != 0 and doc is None
    assert "WORLD_SIZE=2 but --gpus 4" in (proc.stderr + proc.stdout)


@pytest.mark.gpu
def test_two_rank_strong_scaling_reproduces_single_process_histogram():
    """Two ranks (gloo rendezvous, sharing the box's one GPU) split a fixed set of error sets; the
    checksum of the exchanged global histogram equals the single-process one, in complex64."""
    common = ["--workload", "cfg5", "--sets", "600", "--shots", "50", "--scaling", "strong", "--steps", "1",
              "--warmup", "3", "--no-cpu", "--no-e2e", "--no-c128", "--hypersamples", "8"]
    one, doc1 = _run(["--gpus", "1"] + common)
    two, doc2 = _run(["--gpus", "2"] + common, env_extra={"PTSBE_BENCH_BACKEND": "gloo"})
    assert one.returncode == 0, one.stderr[-2000:]
    assert two.returncode == 0, two.stderr[-2000:]
    assert doc1["n_gpus"] == 1 and doc2["n_gpus"] == 2 and doc2["scaling"] == "strong"
    assert doc1["sampled_shots_per_step"] == doc2["sampled_shots_per_step"]
    assert doc1["histogram_checksum"] == doc2["histogram_checksum"]
    assert doc1["stage_events"][0] == 600
