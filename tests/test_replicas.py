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


def test_reference_arm_only_rank0(capsys, monkeypatch):
    import bench
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "1")

    class A:
        config, steps, warmup, gpus, nev_cpu, max_restarts = "cfg1", 1, 1, 2, 0, 100
    bench.run_reference(A())
    assert capsys.readouterr().out == ""


def test_reference_arm_line(capsys, monkeypatch):
    import json
    import bench
    monkeypatch.setenv("RANK", "0")
    monkeypatch.setenv("WORLD_SIZE", "1")

    class A:
        config, steps, warmup, gpus, nev_cpu, max_restarts = "cfg1", 1, 0, 1, 1, 100
    bench.run_reference(A())
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "GFLOP/s" and line["value"] > 0
    assert line["cpu_baseline"]["cores"] == 1 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["time_to_nev_ms"] > 0
