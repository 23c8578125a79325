"""Schedule-model prediction of multi-GPU scaling (VERDICT r01
item 3(d)). Host only: `tinv_model_run` (csrc/model.cu) simulates the exact
exec DAG the planner compiles -- phase groups, work items, priority levels,
per-rank queues, SEND / RECV -- with per-item costs from the executor's job
decomposition, calibrated on the single-B200 measurements:

  block product 128^3 (mainloop)   16.8 us (33.0K cycles at 1965 MHz)
  per-item overhead (epilogue + bookkeeping)     3.2 us (6.3K cycles)
  128-block Cholesky + inverse                   65 us in situ (43.8 us alone: 65K + 21K cycles,
                                                 tools/micro/potrf128.cu; C2's traced POTRFs take 231 us)
  128-block triangular inverse                   10.7 us (21K cycles)
  ready -> start latency of an item              10 us (C2 trace: POTRF -> TRSM gaps 11 us)

  python tools/scaling_model.py [--configs c1,c2,c3] [--ranks 1,2,4,8] [--emulate]

--emulate models the one-launch emulation (148 // N SMs per rank, transfers
through HBM) so it can be checked against tools/emulate_scaling.py's
measurements; without it each rank is a full B200 (148 SMs, NVLink link
latency), the real 8-GPU node.
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1002_4057_b200._native import MODEL_COST as COST  # noqa: E402
CONFIGS = {"c1": (1024, 128, "out", "UDU"), "c2": (8192, 256, "out", "UDU"), "c3": (32768, 512, "out", "UDU"),
           "c5": (65536, 1024, "out", "UDU")}


def model(n, nb, placement, loops, ranks, sms, cost, emulate=False, crit=False):
    import paper_1002_4057_b200 as P
    from paper_1002_4057_b200 import _native
    from paper_1002_4057_b200.distributed import default_grid, distribute, transfer_plan

    t = n // nb
    s = P.gen_inversion(t, P.VariantConfig(P.Placement(placement), loops, True))
    if ranks == 1:
        return _native.model_run(n, nb, s.table(), t, sorted(s.barriers), sms_per_rank=sms, cost=cost, with_crit=crit)
    d = distribute(s, default_grid(ranks))
    table, aux, nrecv, _, who = transfer_plan(d, -1, with_ranks=True)
    per = sms // ranks if emulate else sms
    return _native.model_run(n, nb, table, t, aux=aux, nrecv=nrecv, rank_of=who, nranks=ranks, sms_per_rank=per,
                             cost=cost, with_crit=crit)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3")
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--emulate", action="store_true")
    ap.add_argument("--sms", type=int, default=148)
    ap.add_argument("--cost", default="", help="overrides, e.g. blk=16.5,link=5")
    args = ap.parse_args()
    cost = dict(COST)
    for kv in filter(None, args.cost.split(",")):
        k, v = kv.split("=")
        cost[k] = float(v)
    if args.emulate:
        cost["link"] = 1.0  # flag through HBM, polled by the same GPU
    out = []
    for cfg in args.configs.split(","):
        n, nb, pl, lo = CONFIGS[cfg]
        t1 = None
        for r in [int(x) for x in args.ranks.split(",")]:
            w0 = time.perf_counter()
            mk, busy, crit = model(n, nb, pl, lo, r, args.sms, cost, args.emulate, True)
            if t1 is None:
                t1 = mk
            sms_used = args.sms if r == 1 else (r * (args.sms // r) if args.emulate else r * args.sms)
            eff = t1 * args.sms / (mk * sms_used)
            row = {"config": cfg, "ranks": r, "model_ms": mk / 1e3, "efficiency": eff,
                   "busy_max_over_mean": float(busy.max() / busy.mean()), "sms_used": sms_used,
                   "critical_chain_ms": {k: round(v / 1e3, 2) for k, v in sorted(crit.items(), key=lambda x: -x[1])},
                   "model_s": round(time.perf_counter() - w0, 2)}
            out.append(row)
            print(json.dumps(row), flush=True)
    print(json.dumps({"cost_us": cost, "emulate": args.emulate, "rows": out}))


if __name__ == "__main__":
    main()
