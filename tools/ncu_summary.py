"""Summarise an `ncu --set full` capture (raw page CSV) of the evaluation kernels into the
profiles/*_ncu.json files bench.py reads (dram traffic, executed FP64 flops per pair,
pipe utilisation, stall ratios)."""
import csv
import json
import sys


def summarise(raw_csv, pairs_by_kernel, source):
    rows = list(csv.reader(open(raw_csv)))
    h, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = dict(zip(h, vals))
        f = lambda k: float(d[k])
        name = d.get("Kernel Name", "")
        key = next((k for k in pairs_by_kernel if k in name), None)
        dur = f("gpu__time_duration.sum") * {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}[units[h.index("gpu__time_duration.sum")]]
        clk = f("sm__cycles_elapsed.avg.per_second") * 1e9
        cyc = dur * clk
        dfma = f("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed") * cyc
        dmul = f("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed") * cyc
        dadd = f("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed") * cyc
        flops = 2 * dfma + dmul + dadd
        pairs = pairs_by_kernel.get(key)
        mb = lambda k: f(k) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[h.index(k)]]
        rec = {
            "kernel": name.split("(")[0], "source": source, "duration_ms": dur * 1e3, "sm_clock_ghz": clk / 1e9,
            "dram_bytes_per_launch": mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum"),
            "pair_evals": pairs, "fp64_flops_executed": flops,
            "fp64_flop_per_pair_executed": flops / pairs if pairs else None,
            "fp64_inst_per_pair": (dfma + dmul + dadd) / pairs if pairs else None,
            "fp64_tflops_executed": flops / dur / 1e12,
            "fp64_pipe_active_pct": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "registers_per_thread": f("launch__registers_per_thread"),
            "smem_bank_conflicts": f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
            "warp_instructions": f("smsp__inst_executed.sum"),
            "warp_instructions_per_32_pairs": f("smsp__inst_executed.sum") / (pairs / 32) if pairs else None,
            "stall_ratios_per_issue": {k.split("stalled_")[1].split("_per")[0]: round(f(k), 3) for k in h
                                       if k.startswith("smsp__average_warps_issue_stalled_")
                                       and k.endswith("_per_issue_active.ratio") and f(k) > 0.02},
        }
        out.append(rec)
    return out


if __name__ == "__main__":
    raw, src, outp = sys.argv[1], sys.argv[2], sys.argv[3]
    pairs = json.loads(sys.argv[4])
    res = summarise(raw, pairs, src)
    json.dump(res if len(res) > 1 else res[0], open(outp, "w"), indent=1)
    print(json.dumps(res, indent=1))
