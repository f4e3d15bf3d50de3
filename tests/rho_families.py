"""Planned imbalance rho_s (metrics.hpp:173-186) of every U x R split at G=8 for the
three generator families (mask.hpp:166-228) and seeds 1..N, under the uniform
USP plan (default_plan, metrics.hpp:105-113) and the db-SP plan (plan_dual,
planner.hpp:175-217) -- SURVEY.md §8(d) "report all three families, seeds
1..N".  Host-only (the planner library); the measured-kernel counterpart is
tests/sp_scaling_projection.py wan wan-random wan-banded.
    python tests/rho_families.py [seeds] [workload] > out.json"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2511_23113_b200 as D  # noqa: E402
from paper_2511_23113_b200.workloads import WORKLOADS  # noqa: E402


def main():
    seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    base = WORKLOADS[sys.argv[2] if len(sys.argv) > 2 else "wan"]
    out = {"workload": base.name, "gpus": 8, "seeds": list(range(1, seeds + 1)), "families": {}}
    for fam in ("clustered", "random", "banded"):
        rows = {}
        for seed in range(1, seeds + 1):
            spec = base.spec(seed)
            spec = D.GeneratorSpec(**{**spec.__dict__, "pattern": fam})
            masks = D.generate_mask_set(spec)
            for st in D.enumerate_strategies(8):
                r = rows.setdefault(str(st), {"uniform": [], "dbsp": []})
                r["uniform"].append(D.imbalance_ratio(D.workload_table(masks, st, D.default_plan(masks, st))))
                r["dbsp"].append(D.imbalance_ratio(D.workload_table(masks, st, D.plan_dual(masks, st).plan)))
        summ = {}
        for st, r in rows.items():
            summ[st] = {k: {"mean": round(sum(v) / len(v), 4), "worst": round(max(v), 4)} for k, v in r.items()}
        best_u = min(summ, key=lambda s: summ[s]["uniform"]["mean"])
        best_d = min(summ, key=lambda s: summ[s]["dbsp"]["mean"])
        out["families"][fam] = {"splits": summ, "best_uniform": best_u, "best_dbsp": best_d,
                                "rho_best_uniform": summ[best_u]["uniform"]["mean"],
                                "rho_best_dbsp": summ[best_d]["dbsp"]["mean"]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
