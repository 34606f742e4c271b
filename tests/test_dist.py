"""N > 1 host logic on CPU (gloo, world_size 2): the library's work-unit sharding is a
partition into contiguous blocks; an all-reduce (sum) of disjoint-support chunk-partial arrays
reproduces the single-process array exactly (x + 0 = x), so the ordered double-double finalize
is bit-identical for any rank count.  The GPU kernels are not involved here."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def partial_value(u):
    """A deterministic, 'ugly' double-double partial per unit (stands in for a chunk sum)."""
    rng = np.random.Generator(np.random.PCG64(1000 + u))
    hi = rng.standard_normal(2) * 10.0 ** rng.integers(-8, 8, 2)
    lo = hi * 2.0 ** -60 * rng.standard_normal(2)
    return np.array([hi[0], lo[0], hi[1], lo[1], abs(hi[0]), 0.0, 0.0, 0.0])


def two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def _dd_add(acc, hi2, lo2):
    s, e = two_sum(acc[0], hi2)
    e += acc[1] + lo2
    hi = s + e
    return [hi, e - (hi - s)]


def dd_finalize(P):
    """Python mirror of finalize_kernel's fixed order: 128 contiguous unit ranges are each
    double-double summed in ascending order, then the 128 range sums in ascending order
    (the order depends only on the unit count, not on the number of ranks)."""
    units = P.shape[0]
    c = (units + 127) // 128
    out = []
    for col in (0, 2):
        total = [0.0, 0.0]
        for i in range(128):
            acc = [0.0, 0.0]
            for u in range(min(units, c * i), min(units, c * i + c)):
                acc = _dd_add(acc, P[u, col], P[u, col + 1])
            total = _dd_add(total, acc[0], acc[1])
        out.append(total[0] + total[1])
    return out


def _worker(rank, world, port, units, q):
    import paper_2108_01622_b200 as L
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, e = L.lhaf_shard_units(units, rank, world)
    P = np.zeros((units, 8))
    for u in range(b, e):
        P[u] = partial_value(u)
    t = torch.from_numpy(P)
    dist.all_reduce(t)
    q.put((rank, b, e, t.numpy().tobytes()))
    dist.destroy_process_group()


@pytest.mark.parametrize("units,world", [(37, 2), (8192, 2), (5, 2)])
def test_sharded_partials_allreduce_exact(lib, units, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, units, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    # contiguous partition of [0, units)
    assert res[0][1] == 0 and res[-1][2] == units
    for a, b in zip(res, res[1:]):
        assert a[2] == b[1]
    full = np.stack([partial_value(u) for u in range(units)])
    for _, _, _, buf in res:
        got = np.frombuffer(buf, dtype=np.float64).reshape(units, 8)
        assert np.array_equal(got, full)                 # exact: disjoint support
        assert dd_finalize(got) == dd_finalize(full)    # hence bit-identical finalize


def test_shard_units_partition_many_ranks(lib):
    for units in (1, 7, 32768, 2 ** 35 + 3):
        for R in (1, 2, 3, 4, 8, 16):
            prev = 0
            for r in range(R):
                b, e = lib.lhaf_shard_units(units, r, R)
                assert b == prev and e >= b
                prev = e
            assert prev == units


class _GlooJob:
    """Stand-in for paper_2108_01622_b200.Job with bench.py's per-step calls, on CPU: the
    "kernel" writes each unit's partial (overwriting, as the sieve does), the range all-reduce
    is a gloo all_reduce of that slice, finalize is the ordered double-double sum."""

    def __init__(self, units):
        self.P = torch.zeros((units, 8), dtype=torch.float64)
        self.out = None

    def reset_range(self, b, e, stream=0):
        self.P[b:e] = 0.0

    def run(self, b, e, stream=0):
        for u in range(b, e):
            self.P[u] = torch.from_numpy(partial_value(u))

    def allreduce_range(self, b, e, stream=0):
        view = self.P[b:e].clone()
        dist.all_reduce(view)
        self.P[b:e] = view

    def finalize_dev(self, out_ptr, stream=0):
        self.out = dd_finalize(self.P.numpy())


def _bench_worker(rank, world, port, units, slices, steps, q):
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    job = _GlooJob(units)
    for s in range(steps):
        bench.hot_path_step(job, s, units, slices, rank, world, 0, 0)
    q.put((rank, job.out))
    dist.destroy_process_group()


@pytest.mark.parametrize("units,slices,steps", [(37, 1, 5), (300, 4, 9), (64, 64, 70)])
def test_bench_step_protocol_two_ranks(units, slices, steps):
    # bench.py's step (zero the slice, evaluate the rank's share, all-reduce the slice,
    # finalize) over repeated slices: the 2-rank result equals the 1-rank result bit for bit
    # and nothing is counted twice when a slice is evaluated again (bench.py:254)
    import bench
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_bench_worker, args=(r, 2, port, units, slices, steps, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    covered = set()
    for s in range(steps):
        sb, se, _, _ = bench.slice_bounds(units, s, slices, 0, 1)
        covered.update(range(sb, se))
    P = np.zeros((units, 8))
    for u in covered:
        P[u] = partial_value(u)
    want = dd_finalize(P)
    assert res[0] == want and res[1] == want, (res, want)
