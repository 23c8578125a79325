"""Multi-GPU schedule emulated on ONE B200.

The 2D block-cyclic distributed plan of N ranks (every task on the owner of
its output tile, one SEND / RECV pair per tile version a rank consumes from
another owner) runs in one executor launch with rank r on its own group of
floor(148 / N) SMs and its own priority queues (tinv_plan_create_ranks).
Per-rank busy time comes from the per-CTA idle counters.

Emulated efficiency E_N = T_1 * 148 / (T_N * N * floor(148 / N)): 1.0 means
the distribution (load balance, SEND copies, partitioned scheduling) costs no
SM time over the single-GPU run. It does NOT model the 8x shorter run a real
node would have against the same critical path (see tools/scaling_model.py),
nor NVLink latency (transfers go through HBM here).

  python tools/emulate_scaling.py [--n 32768 --nb 512 --ranks 1,2,4,8 --reps 3]
"""

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--nb", type=int, default=512)
    ap.add_argument("--loops", default="UDU")
    ap.add_argument("--placement", default="out")
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()

    import numpy as np
    import torch

    import paper_1002_4057_b200 as P
    from paper_1002_4057_b200 import _native
    from paper_1002_4057_b200.distributed import default_grid, distribute, transfer_plan

    n, nb = args.n, args.nb
    t = n // nb
    gen = torch.Generator(device="cuda").manual_seed(0)
    g = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=gen)
    a = torch.matmul(g, g.T)
    del g
    a.div_(n)
    a.diagonal().add_(1.0)
    a = torch.tril(a) + torch.tril(a, -1).T
    s = P.gen_inversion(t, P.VariantConfig(P.Placement(args.placement), args.loops, True))
    ctx = _native.Context(n, nb)
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    ref = None
    rows = []
    for N in [int(x) for x in args.ranks.split(",")]:
        grid = default_grid(N)
        if N == 1:
            plan = _native.Plan(ctx, s.table(), t, np.zeros(0, np.int64))
            info = {"transfers": 0, "load_max_over_mean": 1.0}
        else:
            d = distribute(s, grid)
            table, aux, nrecv, src, who = transfer_plan(d, -1, with_ranks=True)
            plan = _native.Plan.ranks(ctx, table, t, aux, nrecv, who, N)
            st = d.stats(nb)
            info = {"transfers": st["transfers"], "load_max_over_mean": st["load_max_over_mean"]}
        assert plan.rc == 0, plan.msg
        ms, busy = [], []
        for _ in range(args.reps):
            ctx.put_dense_device(a.data_ptr(), n)
            rc, err, k = plan.run()
            assert rc == 0, plan.msg
            ms.append(k)
            idle, rank = plan.cta_idle()
            busy.append([float(np.mean(k - idle[rank == r] * 1e-6)) for r in range(N)])
        x = torch.empty_like(a)
        ctx.get_dense_device(x.data_ptr(), n, _native.DENSE_SYMMETRIZE)
        if ref is None:
            ref = x
        bit = bool(torch.equal(x, ref))
        del x
        plan.close()
        med = statistics.median(ms)
        per_rank = np.median(np.array(busy), axis=0)
        sms = nsm if N == 1 else N * (nsm // N)
        rows.append({"ranks": N, "grid": list(grid), "sms_used": sms, "kernel_ms": med,
                     "busy_ms_per_rank": [round(float(b), 2) for b in per_rank],
                     "busy_max_over_mean": float(per_rank.max() / per_rank.mean()),
                     "bitwise_equal_1rank": bit, **info})
        print(json.dumps(rows[-1]), flush=True)
    t1 = rows[0]["kernel_ms"]
    for r in rows:
        r["emulated_efficiency"] = t1 * nsm / (r["kernel_ms"] * r["sms_used"])
    print(json.dumps({"workload": f"n={n}, nb={nb}, {args.placement}-of-place, {args.loops}, pipelined",
                      "rows": rows}))
    ctx.close()


if __name__ == "__main__":
    main()
