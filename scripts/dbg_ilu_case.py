"""Box vs CSR ILU(0) factors on one preset case (dev tool)."""
import sys

import numpy as np

sys.path.insert(0, '.')
from paper_2004_13961_b200 import _lib, make_problem  # noqa: E402
from paper_2004_13961_b200.precond import assemble_M  # noqa: E402
from paper_2004_13961_b200.sparse import IluFactors, SparseMatrix, ilu0  # noqa: E402

case, n = (sys.argv[1], int(sys.argv[2])) if len(sys.argv) > 2 else ("example4a", 40)
spec = make_problem(case, n)
m = assemble_M(spec, (4, 3), 0)
print("n", m.n, "nnz", m.nnz)
csr = SparseMatrix(m.n, m.indptr, m.indices, m.values)
fc = ilu0(csr)
try:
    fb = ilu0(m)
except Exception as e:
    print("box:", e, _lib.load().lp_last_error())
    fb = IluFactors(m, m._handle)
for part in ("L", "U"):
    b, c = getattr(fb, part), getattr(fc, part)
    assert np.array_equal(b.indptr, c.indptr)
    d = b.values != c.values
    rows = np.searchsorted(b.indptr, np.nonzero(d)[0], side="right") - 1
    print(part, "differing entries", d.sum(), "first rows", np.unique(rows)[:10])
