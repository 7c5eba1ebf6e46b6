"""Multi-rank plumbing of bench.py on CPU (gloo, world_size 2): the timings are reduced to
the max over ranks, the whole-job value counts every rank's replica move, and the
reference arm prints only on rank 0.  (The move itself does not shard: "replicas only",
SURVEY 8(e); the GPU path uses the same functions over NCCL.)"""
import os
import socket
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    vals = bench.max_over_ranks([1.0 + rank, 10.0 - rank, 3.5])
    q.put((rank, vals, bench.job_value(world, vals[0])))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, vals, value in out:
        assert vals == [2.0, 10.0, 3.5]            # element-wise max over the two ranks
        assert value == pytest.approx(2 * 1e3 / 2.0)   # both replicas' moves / slowest rank


def test_single_process_passthrough():
    import bench
    assert bench.max_over_ranks([1.5, 2.5]) == [1.5, 2.5]
    assert bench.job_value(1, 4.0) == pytest.approx(250.0)


def test_reference_arm_prints_only_on_rank0(capsys, monkeypatch):
    import bench
    import ctm_inputs as ci

    class A:
        steps, warmup, gpus = 1, 0, 2

    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")
    bench.bench_reference(A, ci.CONFIGS["tiny"])
    assert capsys.readouterr().out == ""
