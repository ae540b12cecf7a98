"""N > 1 launch plumbing of bench.py on CPU (gloo, world_size 2).

The driver launches `bench.py --gpus N` under torch.distributed.run, one
rank per GPU: rank 0 drives the plan's devices and prints the single JSON
line, every rank joins the barriers, the timing is the max over ranks.  The
GPU arm needs CUDA; the reference arm (`--impl reference`, the compiled
reference on the host cores) exercises the same rank / barrier / reporting
path here.
"""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _max_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import bench

    r, w, dist = bench.dist_setup()
    assert (r, w) == (rank, world)
    bench.barrier(dist)
    v = bench.max_over_ranks(dist, float(10 * rank + 1))
    out[rank] = v
    dist.destroy_process_group()


def test_max_over_ranks_gloo():
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_max_worker, args=(2, port, out), nprocs=2, join=True)
        assert out[0] == out[1] == 11.0


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libpipeplan_ref.so")),
                    reason="compiled reference (oracle/_ref) not built")
def test_bench_reference_arm_two_ranks():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--impl", "reference",
           "--workload", "mlp784", "--steps", "1", "--warmup", "3", "--gpus", "2"]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference"
    assert d["e2e"]["h2d_bytes_per_step"] == 0
