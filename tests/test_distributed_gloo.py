"""Multi-process (world_size 2, gloo, CPU) test of the candidate-sharded profiling path: sharding,
all_gather and un-permutation give every rank the same full result vector as a 1-rank run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from workloads import configs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fake_profile(cands):
    """stand-in for mt_profile_batch on CPU: a deterministic 'latency' per candidate and a status
    (infeasible when some stage of the pointer matrix is empty for every tenant)"""
    lat, st = [], []
    for rho in cands:
        key = sum((i + 1) * (k + 3) * v for i, row in enumerate(rho) for k, v in enumerate(row))
        lat.append(100.0 + (key % 997) * 0.5)
        st.append(0 if key % 13 else 2)
    return np.array(lat, np.float32), np.array(st, np.int32)


def _worker(rank, world, port, n, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2111_14255_b200 import distributed as D
    cands = configs.sample_candidates([56, 21, 54], n, seed=14255)
    lat, st = D.profile_distributed(_fake_profile, cands, rank, world)
    out[rank] = (lat.tolist(), st.tolist())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [17, 64])
def test_sharded_profile_gather_gloo_world2(n):
    pytest.importorskip("paper_2111_14255_b200.mt")
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, n, out), nprocs=2, join=True)
        res = dict(out)
    ref_lat, ref_st = _fake_profile(configs.sample_candidates([56, 21, 54], n, seed=14255))
    for r in (0, 1):
        lat, st = res[r]
        np.testing.assert_array_equal(np.array(lat, np.float32), ref_lat)
        np.testing.assert_array_equal(np.array(st, np.int32), ref_st)


def test_shard_indices_partition():
    from paper_2111_14255_b200 import distributed as D
    for n in (0, 1, 7, 1024):
        for w in (1, 2, 3, 8):
            allc = sorted(c for r in range(w) for c in D.shard_indices(n, r, w))
            assert allc == list(range(n))


def _slow_profile(rank):
    """rank r's GPU runs 10 % * r slower than rank 0's"""
    def f(cands):
        lat, st = _fake_profile(cands)
        return lat * (1.0 + 0.1 * rank), st
    return f


def _worker_norm(rank, world, port, n, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2111_14255_b200 import distributed as D
    cands = configs.sample_candidates([56, 21, 54], n, seed=14255)
    info = {}
    lat, st = D.profile_distributed(_slow_profile(rank), cands, rank, world, ref=(0, 1), info=info)
    out[rank] = (lat.tolist(), st.tolist(), info["scales"])
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_profile_per_gpu_normalisation_gloo_world2():
    """ranks with different clocks (rank 1 10 % slower): after scaling by the shared reference
    schedules (the two extremes), every candidate's latency equals the average-GPU latency, so
    candidates measured on different ranks are comparable (SURVEY §7 hard part 5)"""
    pytest.importorskip("paper_2111_14255_b200.mt")
    n = 40
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker_norm, args=(2, port, n, out), nprocs=2, join=True)
        res = dict(out)
    ref_lat, ref_st = _fake_profile(configs.sample_candidates([56, 21, 54], n, seed=14255))
    for r in (0, 1):
        lat, st, scales = res[r]
        np.testing.assert_allclose(scales, [1.05, 1.05 / 1.1], rtol=1e-6)
        np.testing.assert_allclose(np.array(lat), ref_lat * 1.05, rtol=1e-5)
        np.testing.assert_array_equal(np.array(st, np.int32), ref_st)


def _worker_bench(rank, world, port, n, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    L = [56, 21, 54]
    cands = configs.sample_candidates(L, n, seed=14255)
    res = bench.profiling_leg(_fake_profile, cands, L, rank, world, cd_p=(0, 1, 2), cd_m=4)
    out[rank] = (res["lat"].tolist(), res["st"].tolist(), res["cd"]["best_us"], res["cd"]["evaluations"],
                 res["cd"]["best_P"])
    dist.barrier()
    dist.destroy_process_group()


def test_bench_profiling_leg_multirank_gloo_world2():
    """bench.py's multi-rank profiling code path (sharded profiling + distributed coordinate
    descent over P, one gather per (round, row)) with a stand-in profiler: every rank ends with
    the 1-rank result, so the N-GPU bench line is the same computation spread over N GPUs"""
    import bench
    n = 48
    L = [56, 21, 54]
    one = bench.profiling_leg(_fake_profile, configs.sample_candidates(L, n, seed=14255), L, 0, 1,
                              cd_p=(0, 1, 2), cd_m=4)
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker_bench, args=(2, port, n, out), nprocs=2, join=True)
        res = dict(out)
    for r in (0, 1):
        lat, st, best, ev, bp = res[r]
        np.testing.assert_array_equal(np.array(lat, np.float32), one["lat"])
        np.testing.assert_array_equal(np.array(st, np.int32), one["st"])
        assert best == one["cd"]["best_us"] and ev == one["cd"]["evaluations"] and bp == one["cd"]["best_P"]
    assert one["cd"]["evaluations"] == 1 + 2 * (1 + 3 * 4)


def test_bench_spawns_torchrun_for_multi_gpu():
    """--gpus N > 1 without WORLD_SIZE re-launches bench.py under torch.distributed.run (the
    driver's own launch line), so n_gpus reports the ranks"""
    import bench
    cmd = bench.torchrun_cmd(8, ["--gpus", "8", "--steps", "5"], 29555)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "8", "--steps", "5"]
    assert cmd[cmd.index("--master-port") + 1] == "29555"
