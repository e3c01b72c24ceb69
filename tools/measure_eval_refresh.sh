# Refresh the evaluation-kernel ncu summary (the file bench.py's roofline reads, keyed by the
# evaluation sources' hash) after an evaluation-source edit, then the bench line that uses
# it and the GPU tests.  Usage (under gpurun): bash tools/measure_eval_refresh.sh TAG
T=${1:-r02}
mkdir -p gpurun_out
# pair-evaluation counts for the summary (its roofline is refused until the capture exists)
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^k_mutual$" -c 1 -o gpurun_out/prof_${T}_mut python tools/prof_once.py c5 > gpurun_out/ncu_mut_$T.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:"^k_interact$" -c 1 -o gpurun_out/prof_${T}_int python tools/prof_once.py c5 > gpurun_out/ncu_int_$T.log 2>&1
for r in mut int; do ncu -i gpurun_out/prof_${T}_$r.ncu-rep --page raw --csv > gpurun_out/prof_${T}_$r.csv 2>/dev/null; done
python tools/ncu_eval_summary.py $T > gpurun_out/ncu_eval_summary_$T.log 2>&1
cp gpurun_out/ncu_eval_summary_$T.json profiles/r02_interact_sal_ncu.json  # the box's copy: the bench reads it
timeout 600 python bench.py > gpurun_out/bench_final_$T.json 2> gpurun_out/bench_final_$T.err
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_all_$T.log 2>&1; echo "rc $?" >> gpurun_out/pytest_all_$T.log
echo done
