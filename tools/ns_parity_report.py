"""Per-component max error of the device NS RHS against the C oracle
(oracle/ns_oracle.c), relative to each field's max, at a few sizes: the
numbers DESIGN.md quotes for the single-RHS parity."""
import sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import numpy as np
import paper_1309_7327_b200 as P
from paper_1309_7327_b200 import workloads as W
from oracle import oracle as O

DX = 1e-4
for n, kw in ((16, {}), (24, {"hot_spot": True}), (32, {}), (32, {"ignition": True})):
    T, p, uvw, Y = W.ns_primitives(n, **kw)
    U = O.ns_conserved(T, p, uvw, Y)
    op = P.NsOperator(n, n, n, DX)
    for part, name in ((P.NS_FULL, "full"), (P.NS_ADVDIFF, "advdiff"), (P.NS_CHEM, "chem")):
        ref = O.ns_rhs(U, DX, part)
        got = (op.full, op.advdiff, op.chem)[part](0.0, U)
        err = [float(np.abs(got[v] - ref[v]).max() / max(np.abs(ref[v]).max(), 1e-300))
               for v in range(ref.shape[0])]
        print(f"{n}^3 {kw} {name}: max rel err {max(err):.2e} (component {int(np.argmax(err))})")
