# Late round-2 re-measurement after an evaluation-source edit (under gpurun, one B200):
# the evaluation-kernel ncu captures first (bench.py refuses a capture whose source hash
# differs), then the bench line, the launch list, the GPU tests + smoke, per-config phases,
# the BVE step, CSTC and the emulated scaling.  Usage: bash tools/measure_r02_late.sh TAG
T=${1:-r02l}
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$T.json 2> gpurun_out/bench_pre_$T.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^k_mutual$" -c 1 -o gpurun_out/prof_${T}_mut python tools/prof_once.py c5 > gpurun_out/ncu_mut_$T.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:"^k_interact$" -c 1 -o gpurun_out/prof_${T}_int python tools/prof_once.py c5 > gpurun_out/ncu_int_$T.log 2>&1
for r in mut int; do ncu -i gpurun_out/prof_${T}_$r.ncu-rep --page raw --csv > gpurun_out/prof_${T}_$r.csv 2>/dev/null; done
python tools/ncu_eval_summary.py $T > gpurun_out/ncu_eval_summary_$T.log 2>&1
cp gpurun_out/ncu_eval_summary_$T.json profiles/r02_interact_sal_ncu.json
timeout 600 python bench.py > gpurun_out/bench_final_$T.json 2> gpurun_out/bench_final_$T.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$T.log 2>&1
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_all_$T.log 2>&1; echo "rc $?" >> gpurun_out/pytest_all_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "rc $?" >> gpurun_out/smoke_$T.log
for c in c2 c3 c5; do TREE_MODES=sort timeout 300 python tools/tree_perf.py $c 5; done > gpurun_out/phases_${T}.txt 2>&1
timeout 1200 python tools/bve_perf.py 9 > gpurun_out/bve_$T.log 2>&1
timeout 1500 python tools/cstc_perf.py c2 c3 c5 > gpurun_out/cstc_$T.log 2>&1
timeout 900 python tools/scaling_emulation.py c5 gpurun_out/scaling_${T}.json > gpurun_out/scaling_${T}.log 2>&1
# the reference arm, the HBM-kernel ncu pass (every non-evaluation kernel) and the full-size parity run
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size
timeout 900 ncu --metrics $M --clock-control none -k "regex:^(?!k_interact|k_mutual|k_dfma).*" --csv --log-file gpurun_out/hbm_$T.csv python tools/prof_once.py c5 > gpurun_out/hbm_$T.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -s > gpurun_out/parity_fullsize_$T.log 2>&1
rm -f gpurun_out/*.ncu-rep  # the raw-page CSVs are kept; the reports would pass gpurun's 64 MiB return limit
echo done
# then here: cp the outputs over profiles/r02_* (profiles/README.md lists them), python tools/launch_summary.py
# gpurun_out/launches_$T.csv profiles/r02_launches_c5_step_summary.json, python tools/ncu_hbm_summary.py
# gpurun_out/hbm_$T.csv profiles/r02_hbm_kernels_ncu.json
