"""GPU: the NS kernels converge to the exact manufactured-solution RHS
(tests/ns_mms.py, symbolic calculus of PAPER.md:143-213, :399-428) at
eighth order, like the oracle (test_ns_mms.py), and agree with the oracle at
every grid to <= 1e-10 of each field's max."""
import numpy as np
import pytest

import ns_mms as M
import paper_1309_7327_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu
NS = (32, 48, 64)


def _percomp(a, b):
    return max(float(np.abs(a[v] - b[v]).max() / np.abs(b[v]).max()) for v in range(a.shape[0]))


@pytest.mark.parametrize("part", [P.NS_FULL, P.NS_ADVDIFF])
def test_gpu_converges_to_exact_rhs(cuda, part):
    O.set_threads(0)
    errs = []
    for n in NS:
        U, ex, dx = M.evaluate(n)
        exact = sum(v for k, v in ex.items() if part == P.NS_FULL or k != "chem")
        op = P.NsOperator(n, n, n, dx)
        got = (op.full if part == P.NS_FULL else op.advdiff)(0.0, U)
        errs.append(M.term_error(got, exact))
        assert _percomp(got, O.ns_rhs(U, dx, part)) <= 1e-10
    slope = np.log(errs[-2] / errs[-1]) / np.log(NS[-1] / NS[-2])
    assert abs(slope - 8.0) <= 0.3, (errs, slope)
