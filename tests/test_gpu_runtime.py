"""GPU tests of the runtime around the kernels: the NCCL exchange step (S8(e) a12)
through a real communicator, slice-wise evaluation as bench.py does it, and the device-pointer
entry point's stream ordering."""
import os

import numpy as np
import pytest

import gbs_inputs as G

pytestmark = pytest.mark.gpu


def test_nccl_one_rank_allreduce_bit_identical(lib):
    # lhaf_init_rank(0, 1, id) creates a one-rank NCCL communicator, so lhaf_job_allreduce runs
    # ncclAllReduce exactly as it does with N ranks; the result must be bit-identical to the
    # no-communicator path (x + 0 = x over disjoint unit supports)
    cfg = G.config(3)
    job = lib.Job(cfg["A"], cfg["gamma"], cfg["reps"])
    job.reset(); job.run(); job.allreduce()
    plain = job.finalize()[0]
    uid = lib.lhaf_get_unique_id()
    lib.lhaf_init_rank(0, 1, uid, 0)
    try:
        assert lib.lhaf_rank_info() == (0, 1)
        job.reset(); job.run(); job.allreduce()
        via_nccl = job.finalize()[0]
        # slice-wise: zero a slice, run it, all-reduce just that slice (bench.py's step)
        U = job.units
        job.reset()
        for s in range(4):
            b, e = U * s // 4, U * (s + 1) // 4
            job.reset_range(b, e)
            job.run(b, e)
            job.allreduce_range(b, e)
        sliced = job.finalize()[0]
        # re-running a slice after zeroing it must not double count
        job.reset_range(0, U // 4); job.run(0, U // 4); job.allreduce_range(0, U // 4)
        again = job.finalize()[0]
    finally:
        lib.lhaf_shutdown()
        job.close()
    assert via_nccl == plain and sliced == plain and again == plain, (plain, via_nccl, sliced, again)
    assert lib.lhaf_rank_info() == (0, 1)


def test_batch_dev_orders_after_side_stream(lib, orc):
    # inputs written on a torch side stream, then lhaf_rpt_batch_dev on that stream: the call
    # must see the finished inputs (it synchronises the device before reading them)
    torch = pytest.importorskip("torch")
    rng = G.rng_for(4711)
    k = 8
    A = G.pure_B(G.haar_unitary(k, rng), 0.7)
    g = G.complex_gaussian(k, 0.3, rng)
    reps = np.array([[1, 2, 0, 1, 1, 0, 2, 1], [2, 0, 1, 1, 0, 1, 1, 0]], np.int32)
    side = torch.cuda.Stream()
    At = torch.zeros((k, k), dtype=torch.complex128, device="cuda")
    gt = torch.zeros(k, dtype=torch.complex128, device="cuda")
    out = torch.zeros(4, dtype=torch.float64, device="cuda")
    src_A = torch.from_numpy(A).pin_memory()
    src_g = torch.from_numpy(g).pin_memory()
    with torch.cuda.stream(side):
        torch.cuda._sleep(50_000_000)                   # keep the side stream busy (~25 ms)
        At.copy_(src_A, non_blocking=True)
        gt.copy_(src_g, non_blocking=True)
        lib.lhaf_rpt_batch_dev(At.data_ptr(), gt.data_ptr(), 0, reps, mixed=0,
                               out_dev_ptr=out.data_ptr(), stream_ptr=side.cuda_stream)
    side.synchronize()
    got = out.cpu().numpy()
    for b in range(2):
        ref = orc.lhaf(A, g, reps[b])
        v = complex(got[2 * b], got[2 * b + 1])
        assert abs(v - ref) <= 1e-10 * abs(ref), (b, v, ref)
