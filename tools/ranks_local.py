"""The multi-process runtime's data path with W ranks in one process on one
B200 (distributed.execute_ranks_local at bench scale): per rank a partitioned
store (its own tiles + receive tiles), its transfer plan, its executor on
148/W SMs; all ranks run concurrently, SENDs write into the peers' stores.
Prints per-rank device ms and store bytes next to the one-store run."""
import json
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1002_4057_b200 as P  # noqa: E402
from paper_1002_4057_b200 import _native  # noqa: E402
from paper_1002_4057_b200.distributed import default_grid, distribute, owned_tiles, transfer_plan  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 512
worlds = [int(w) for w in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 2, 4, 8]
t = n // nb
g = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
a = g @ g.T / n
a.diagonal().add_(1.0)
del g
torch.cuda.synchronize()
s = P.gen_inversion(t, P.VariantConfig(P.Placement.OUT_OF_PLACE, "UDU", True))
nsm_all = torch.cuda.get_device_properties(0).multi_processor_count
rows = []
ref_x = None
for W in worlds:
    grid = default_grid(W)
    d = distribute(s, grid)
    ctxs, plans = [], []
    for r in range(W):
        ctx = _native.Context.owned(n, nb, owned_tiles(t, grid, r)) if W > 1 else _native.Context(n, nb)
        ctx.set_sms(nsm_all // W)
        if W > 1:
            table, aux, nrecv, _ = transfer_plan(d, r)
            plan = _native.Plan.xfer(ctx, table, t, aux, nrecv)
        else:
            plan = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64))
        assert plan.rc == 0, plan.msg
        plan.ipc_export()
        ctxs.append(ctx)
        plans.append(plan)
    for r, ctx in enumerate(ctxs):
        ctx.peer_attach(r, ctxs)
    best = None
    for rep in range(2):
        for ctx in ctxs:
            ctx.put_dense_device(a.data_ptr(), n)
            ctx.ipc_reset()
        res = [None] * W
        bar = threading.Barrier(W)

        def run(r):
            bar.wait()
            res[r] = plans[r].run()

        th = [threading.Thread(target=run, args=(r,)) for r in range(W)]
        [x.start() for x in th]
        [x.join() for x in th]
        assert all(x[0] == 0 for x in res), [p.msg for p in plans]
        ms = [x[2] for x in res]
        if best is None or max(ms) < max(best):
            best = ms
    # gather every rank's owned tiles and compare with the one-store result
    x = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    for r, ctx in enumerate(ctxs):
        y = torch.zeros_like(x)
        torch.cuda.synchronize()  # the zero fill (torch's stream) before the gather (the context's stream)
        ctx.get_dense_device(y.data_ptr(), n, _native.DENSE_LOWER)
        torch.cuda.synchronize()
        own = torch.from_numpy(owned_tiles(t, grid, r)).cuda().to(torch.float64)
        x += y * own.repeat_interleave(nb, 0).repeat_interleave(nb, 1)
        del y
    diff = None
    if ref_x is None:
        ref_x = x
        same = True
    else:
        same = bool(torch.equal(x, ref_x))
        if not same:
            dm = (x != ref_x)
            tiles = dm.reshape(t, nb, t, nb).any(dim=3).any(dim=1).nonzero().tolist()
            diff = {"max_abs": float((x - ref_x).abs().max()), "n_diff": int(dm.sum()), "nan": int(x.isnan().sum()),
                    "tiles": tiles[:12], "n_tiles": len(tiles)}
    st = d.stats(nb)
    row = {"ranks": W, "grid": list(grid), "sms_per_rank": nsm_all // W, "rank_ms": [round(v, 2) for v in best],
           "max_ms": round(max(best), 2), "store_gb_per_rank": [round(c.store_bytes() / 1e9, 2) for c in ctxs],
           "full_store_gb": round(2 * t * (t + 1) / 2 * (-(-nb // 128) * 128) ** 2 * 8 / 1e9, 2),
           "transfers": st["transfers"], "bitwise_equal_1rank": same, "diff": diff,
           "emulated_efficiency": round(rows[0]["max_ms"] / max(best), 3) if rows else 1.0}
    rows.append(row)
    print(json.dumps(row), flush=True)
    for p in plans:
        p.close()
    for c in ctxs:
        c.close()
    del x
    torch.cuda.empty_cache()
