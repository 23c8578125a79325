"""Tiny runs of both engines for compute-sanitizer (one tool per call)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1002_4057_b200 as P  # noqa: E402
from oracle import tileinv_oracle as O  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "fused"
if which == "fused":
    a = np.stack([O.spd_matrix(n, s, 0.5) for s, n in enumerate([256] * 3)])
    x = P.invert_batched(a, 256, engine="fused")
    b = np.stack([O.spd_matrix(100, 7, 0.5)] * 2)
    y = P.invert_batched(b, 100, engine="fused")
    print("fused ok", float(np.abs(x[0] @ a[0] - np.eye(256)).max()), float(np.abs(y[0] @ b[0] - np.eye(100)).max()))
else:
    a = O.spd_matrix(512, 0, 1.0)
    x = P.invert(a, 128, P.VariantConfig(P.Placement.OUT_OF_PLACE, "UDU", True))
    print("dag ok", float(np.abs(x @ a - np.eye(512)).max()))
