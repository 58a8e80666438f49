"""Golden Algorithm-1 plan for GPT-3-96 on 64 simulated GPUs from the LIVE reference,
at a size the reference finishes in minutes (1 GiB granularity, batch sizes 8..64):

    python tests/golden/make_golden_gpt.py        (build container only)

The 1 MiB / all-batch-size search of BASELINE config 4 takes the reference hours
(SURVEY.md §6); its device result is checked stage by stage against the oracle
instead (tests/test_gpu_parity.py, tests/test_gpu_gpt_full.py).
"""

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import parapilot as R                                      # noqa: E402
from parapilot import planner as RP                        # noqa: E402

from paper_2307_02031_b200 import workloads as W           # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    c = W.config("gpt")
    model = R.load_model_spec(c.model.to_document())
    cluster = R.load_cluster_spec(c.cluster.to_document())
    opts = RP.PlannerOptions(granularity_bytes=1 << 30, max_batch=64)
    t0 = time.time()
    plan = RP.plan_full(model, cluster, R.CostProfile(), opts)
    dt = time.time() - t0
    doc = {"opts": {"granularity_bytes": 1 << 30, "max_batch": 64}, "ref_seconds": round(dt, 1),
           "plan": {"doc": plan.to_document(), "time_hex": plan.predicted_time_s.hex(),
                    "thr_hex": plan.predicted_throughput.hex(),
                    "alpha": [plan.balance.alpha_t.hex(), plan.balance.alpha_m.hex()],
                    "peaks": [x.hex() for x in plan.peak_mem_per_stage],
                    "strategies": [s.to_string() for s in plan.strategies]}}
    (OUT / "gpt_base.json").write_text(json.dumps(doc, separators=(",", ":")))
    print(f"gpt plan_full (1 GiB, B<=64): {dt:.1f}s  B={plan.batch_size} P={plan.pp_degree}")


if __name__ == "__main__":
    main()
