"""Multi-GPU = replicas only: the host-side plumbing of bench.py
(gloo rendezvous, barrier, max-over-ranks timing, whole-job aggregation) on
world_size 2, CPU only."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ.update({"RANK": str(rank), "WORLD_SIZE": str(ws), "LOCAL_RANK": str(rank),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    import bench
    r, w, local = bench.dist_init()
    bench.barrier(w)
    # each replica measured a different step time; the job time is the max
    mx = bench.allreduce_max(1.0 + rank, w)
    q.put((r, w, local, mx))
    import torch.distributed as dist
    dist.destroy_process_group()


def test_two_replicas_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out == [(0, 2, 0, 2.0), (1, 2, 1, 2.0)]


class _Args:
    config, steps, warmup, gpus, max_restarts = "cfg1", 2, 3, 1, 100
    ref_budget_s, cpu_step_split = 30.0, 1


def test_reference_arm_only_rank0(capsys, monkeypatch):
    import bench
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "1")
    bench.run_reference(_Args())
    assert capsys.readouterr().out == ""


def test_reference_arm_line(capsys, monkeypatch):
    import json
    import bench
    monkeypatch.setenv("RANK", "0")
    monkeypatch.setenv("WORLD_SIZE", "1")
    bench.run_reference(_Args())
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "GFLOP/s" and line["value"] > 0
    assert line["cpu_baseline"]["cores"] >= 1 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["config"]["workload"] == "cfg1" and line["steps"] == 2
    assert set(line["cpu_step_ms"]) == {"spmv", "solve", "cgs2", "other", "total"}


def test_reference_arm_never_loads_the_product():
    """The reference arm takes its pencil from the reference's own spaces code
    (oracle/ref_assembly.cpp): librq_b200.so is never mapped."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.argv=['bench.py','--impl','reference','--config','cfg1','--steps','1',"
            "'--cpu-step-split','0']; import bench; bench.main(); "
            "maps=open('/proc/self/maps').read(); assert 'librq_b200' not in maps, 'product mapped'; "
            "assert 'liboracle' in maps; print('MAPS_OK')")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300,
                         env={**os.environ, "RANK": "0", "WORLD_SIZE": "1"})
    assert out.returncode == 0, out.stderr[-2000:]
    assert "MAPS_OK" in out.stdout and '"impl": "reference"' in out.stdout


def test_gpus_flag_spawns_replicas():
    """`bench.py --gpus 2` without a launcher re-executes itself under
    torch.distributed.run (2 processes): rank 0 prints one line, rank 1 none."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--config", "cfg1",
                          "--steps", "1", "--cpu-step-split", "0"], cwd=root, capture_output=True, text=True,
                         timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and '"n_gpus": 2' in lines[0]
