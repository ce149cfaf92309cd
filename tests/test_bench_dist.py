"""N>1 host logic of bench.py on CPU: world_size-2 gloo process group.

The GPU bench runs one independent replica per rank (weak scaling, no data
collective); the only cross-rank step is the reduction of the timed region
(max over ranks) and of the work (sum over ranks), and the reference arm runs
on rank 0 only.  Both are exercised here without a GPU."""
import os
import socket
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        elapsed, work = bench.job_totals(dist, elapsed=[10.0, 25.0][rank], work=[1.0e6, 3.0e6][rank])
        out[rank] = (elapsed, work)
        # the reference arm: ranks other than 0 exit 0 without work
        if rank != 0:
            class A:
                config = "c1"
                steps = 1
                warmup = 0
                gpus = 2
                ref_threads = 1
            out[world + rank] = bench.run_reference(A())
    finally:
        dist.destroy_process_group()


def test_job_totals_and_reference_ranks_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        assert out[r] == (25.0, 4.0e6)  # slowest rank's time, summed work
    assert out[world + 1] == 0


def test_job_totals_single_process():
    import bench
    assert bench.job_totals(None, 3.0, 7.0) == (3.0, 7.0)


def test_gpus_flag_relaunches_as_ranks():
    """`bench.py --gpus 2` without a rank environment re-launches itself
    through torch.distributed.run; the reference arm then runs on rank 0
    only and prints exactly one JSON line (CPU only: c1, the reference's own
    assembly and solver)."""
    import json
    import subprocess
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--config", "c1", "--steps", "1", "--warmup", "0", "--ref-threads", "2"],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
    assert line["details"]["system"].startswith("reference assemble_monolithic")


def test_launcher_command():
    import bench

    class A:
        gpus = 4
    cmd = bench.launcher_cmd(A(), 12345)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=12345" in cmd
