"""Alternative kernel instantiations against the oracle, each in its own process (the choice
is read once per process from LHAF_V3_ALT): 0 = default (phased reduction), 3 = single-phase
reduction (a second rounding order of the same method), and the v5 kernel (LHAF_KERNEL=5: a
different data layout of the reduction, the third independent code).  Block-diagonal
matrices with the pairs straddling the blocks: lhaf(A1 (+) A2) = lhaf(A1) lhaf(A2),
each factor by the oracle's ET tier."""
import json
import os
import subprocess
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _variant_cases as VC  # noqa: E402

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def refs(orc):
    out = []
    for c in VC.cases():
        A1, g1, A2, g2 = c["blocks"]
        one = [1] * A1.shape[0]
        out.append(orc.lhaf(A1, g1, one, method="et") * orc.lhaf(A2, g2, one, method="et"))
    return out


@pytest.mark.parametrize("alt", [0, 3, "v5", "tree"])
def test_variant_block_diagonal(lib, refs, alt):
    env = (dict(os.environ, LHAF_KERNEL="5") if alt == "v5" else dict(os.environ, LHAF_KERNEL="6")
           if alt == "tree" else dict(os.environ, LHAF_V3_ALT=str(alt), LHAF_KERNEL="3"))
    r = subprocess.run([sys.executable, os.path.join(HERE, "_variant_worker.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = [complex(a, b) for a, b in json.loads(r.stdout.strip().splitlines()[-1])]
    for g, w in zip(got, refs):
        assert abs(g - w) / abs(w) <= 1e-8, (alt, g, w)


def test_v5_zero_weight_deletion_wide(lib):
    # v5 deletes zero-weight indices per term through a warp's compaction buffer; at a
    # bordered size E0 >= 49 the tile has 7-8 positions per lane (the buffer row must hold 64).
    # d = 48: 46 single modes + 2 modes of count 2 (one pair with eta = 2: weight 0 at k = 1);
    # inclusion/exclusion at N = 48 deletes up to every pair.  Both against the tree (the
    # oracle-pinned default path, tests/test_gpu_tree.py) on a Haar GBS instance (tanh r = 0.9).
    import gbs_inputs as G
    import numpy as np
    rng = G.rng_for(4848)
    U = G.haar_unitary(60, rng)
    B = G.pure_B(U, 0.9)[:48, :48]
    g = G.complex_gaussian(48, 0.1, rng)
    reps = np.ones(48, np.int32)
    reps[[5, 17]] = 2
    reps[[40, 41]] = 0
    try:
        lib.lhaf_set_kernel(6)
        ref = lib.lhaf_rpt(B, g, reps)
        ref_et = lib.lhaf_rpt_et(B, g, np.ones(48, np.int32))
        lib.lhaf_set_kernel(5)
        got = lib.lhaf_rpt(B, g, reps)
        got_et = lib.lhaf_rpt_et(B, g, np.ones(48, np.int32))
    finally:
        lib.lhaf_set_kernel(0)
    assert abs(got - ref) / abs(ref) <= 1e-8, (got, ref)
    # ET's own cancellation (Fig. 5): the two ET codes agree far inside 1e-2
    assert abs(got_et - ref_et) / abs(ref_et) <= 1e-2, (got_et, ref_et)
