"""The N > 1 path of bench.py on CPU (gloo, world_size 2; DESIGN.md §7 "replicas only").

The decomposition does not shard (one global argmax per selection), so N
GPUs run N independent replicas and the only cross-rank work is the aggregation of the
timed regions (max over ranks) and of the processed selections (sum over ranks).  These
tests run that aggregation over a real gloo process group, and the reference arm under
torchrun (rank 0 alone runs the oracle, the other ranks exit 0 without work).
"""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch.multiprocessing as tmp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        # rank r: timed regions 10+r and 5-r ms, 1000*(r+1) and 7 selections
        t, c = bench.aggregate([10.0 + rank, 5.0 - rank], [1000 * (rank + 1), 7], world)
        q.put((rank, t, c))
    finally:
        dist.destroy_process_group()


def test_aggregate_gloo_world2():
    world, port = 2, _free_port()
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, t, c in out:
        assert t == [11.0, 5.0]            # max over ranks
        assert c == [3000.0, 14.0]         # sum over ranks
    # whole-job value as bench.py reports it: all ranks' selections / the slowest rank's time
    assert 3000.0 / (11.0 * 1e-3) == pytest.approx(272727.27, rel=1e-6)


def test_aggregate_single_rank_is_identity():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.aggregate([3.5], [12], 1) == ([3.5], [12.0])


def test_reference_arm_under_torchrun_world2():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           "bench.py", "--impl", "reference", "--gpus", "2", "--config", "C0", "--steps", "1", "--warmup", "0"]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1                 # rank 0 alone prints
    ln = lines[0]
    assert ln["impl"] == "reference" and ln["n_gpus"] == 2
    assert ln["value"] > 0 and ln["cpu_baseline"]["kind"] == "oracle"
    assert ln["e2e"]["h2d_bytes_per_step"] == 0
