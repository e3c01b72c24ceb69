"""Combine the `ncu --set full` captures of the two evaluation kernels (tools/measure_round.sh
TAG: gpurun_out/prof_TAG_{mut,int}.csv) into the profiles/*interact_sal_ncu.json summary
bench.py reads.  The per-kernel evaluation counts come from the bench line of the same
run: with L list evaluations and E executed ones, k_mutual executes L - E (each one serves
two list entries) and k_interact 2E - L.

    python tools/ncu_eval_summary.py TAG [out.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from ncu_summary import summarise  # noqa: E402

from paper_2508_13550_b200.srchash import eval_kernel_sha256  # noqa: E402


def main(tag, out):
    bench = json.loads(open(f"gpurun_out/bench_{tag}.json").read().strip().splitlines()[-1])
    L = bench["roofline"]["list_pair_evals_per_launch"]
    E = bench["roofline"]["executed_pair_evals_per_launch"]
    pm, pi = L - E, 2 * E - L
    ks = summarise(f"gpurun_out/prof_{tag}_mut.csv", {"k_mutual": pm}, f"ncu --set full (prof_{tag}_mut, kernel replay)")
    ks += summarise(f"gpurun_out/prof_{tag}_int.csv", {"k_interact": pi},
                    f"ncu --set full (prof_{tag}_int, application replay: kernel replay of its work-queue counter "
                    "returns NaN metrics)")
    dur = sum(k["duration_ms"] for k in ks)
    fl = sum(k["fp64_flops_executed"] for k in ks)
    pe = pm + pi
    res = {"kernel": "evaluation phase: k_mutual<OpSal> (symmetric PP + CC pairs) + k_interact<OpSal> (other PP, CP, CC)",
           "workload": bench["config"]["workload"], "source": f"tools/measure_round.sh {tag}",
           "pair_evals": pe, "duration_ms": dur,
           "dram_bytes_per_launch": sum(k["dram_bytes_per_launch"] for k in ks),
           "fp64_flops_executed": fl, "fp64_flop_per_pair_executed": fl / pe,
           "fp64_inst_per_pair": sum(k["fp64_inst_per_pair"] * k["pair_evals"] for k in ks) / pe,
           "fp64_tflops_executed": fl / dur / 1e9,
           "fp64_pipe_active_pct": sum(k["fp64_pipe_active_pct"] * k["duration_ms"] for k in ks) / dur,
           "source_sha256": eval_kernel_sha256(),
           "kernels": ks}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "kernels"}))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else f"gpurun_out/ncu_eval_summary_{sys.argv[1]}.json")
