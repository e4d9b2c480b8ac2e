"""CPU: the NS oracle pinned against an independent exact solution.

tests/ns_mms.py builds the exact right-hand side of PAPER.md:143-213 (with
the correction velocity of :399-428) for a smooth manufactured periodic state
by symbolic calculus.  The oracle (oracle/ns_oracle.c) must converge to it at
eighth order, term by term: hyperbolic fluxes, viscous stress (momentum and
energy), heat conduction, species diffusion with V_c, enthalpy flux; the
pointwise chemistry must agree to rounding.  The slope band is the
reference's own (pde_test.cpp:135-161: 8 +- 0.3), fitted on the two finest
grids (32^3 is pre-asymptotic for the hyperbolic term, slope 7.74)."""
import numpy as np
import pytest

import ns_mms as M
from oracle import oracle as O

NS = (32, 48, 64)


@pytest.fixture(scope="module")
def errors():
    O.set_threads(0)
    out = {nm: [] for nm in M.TERMS}
    for n in NS:
        U, ex, dx = M.evaluate(n)
        for nm, bit in M.TERMS.items():
            out[nm].append(M.term_error(O.ns_rhs_terms(U, dx, bit), ex[nm]))
        out.setdefault("total", []).append(M.term_error(O.ns_rhs(U, dx, 0), sum(ex.values())))
    return out


@pytest.mark.parametrize("term", ["hyp", "visc", "heat", "spec", "enth", "total"])
def test_oracle_converges_at_eighth_order(errors, term):
    e = errors[term]
    assert all(a > b for a, b in zip(e, e[1:])), e
    slope = np.log(e[-2] / e[-1]) / np.log(NS[-1] / NS[-2])
    assert abs(slope - 8.0) <= 0.3, (term, e, slope)
    assert e[-1] <= 1e-8, e


def test_oracle_chemistry_is_exact_to_rounding(errors):
    assert max(errors["chem"]) <= 1e-13, errors["chem"]
    U, ex, dx = M.evaluate(16, "hot")
    chem = O.ns_rhs_terms(U, dx, M.CHEM)
    assert M.term_error(chem, ex["chem"]) <= 1e-12


def test_terms_add_up_to_the_full_rhs():
    """The term mask splits the full RHS: the sum of the six parts equals it
    to rounding (the full RHS sums in a fixed order)."""
    U, ex, dx = M.evaluate(16)
    full = O.ns_rhs(U, dx, 0)
    parts = sum(O.ns_rhs_terms(U, dx, bit) for bit in M.TERMS.values())
    assert M.term_error(parts, full) <= 1e-12
