"""bench.py's multi-rank plumbing on CPU: torchrun with world_size 2 and the
gloo backend (`bench.py --dry-run`): process group, NCCL-id broadcast, the
partition_scanlines strips (executor.hpp:189-208) and the max-over-ranks
reduction the N-GPU line is timed with.  No kernel is launched."""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_dry_run_two_ranks():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--dry-run"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["dry_run"] and d["n_gpus"] == 2
    assert d["strips"] == [[0, 8192], [8192, 16384]]  # C3 weak scaling: 8192 rows per rank
    assert len(d["id_prefixes"]) == 1  # every rank got rank 0's communicator id
    assert d["max_over_ranks"] == 2.0
    assert d["config"]["parallelism"] == "row-strips2"


def test_bench_dry_run_single():
    r = subprocess.run([sys.executable, "bench.py", "--dry-run", "--config", "c4"], cwd=ROOT, capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["strips"] == [[0, 32768]] and d["bytes_per_cell"] == 48
