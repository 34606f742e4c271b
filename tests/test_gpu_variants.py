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
