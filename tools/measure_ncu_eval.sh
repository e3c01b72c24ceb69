# ncu --set full of the two evaluation kernels at C5 for the current build, summarised into
# profiles/<TAG>_interact_sal_ncu.json (the file bench.py's roofline reads; it carries the
# evaluation kernels' source hash).  Usage (under gpurun): bash tools/measure_ncu_eval.sh TAG
T=${1:-r02}
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^k_mutual$" -c 1 -o gpurun_out/prof_${T}_mut python tools/prof_once.py c5 > gpurun_out/ncu_mut_$T.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:"^k_interact$" -c 1 -o gpurun_out/prof_${T}_int python tools/prof_once.py c5 > gpurun_out/ncu_int_$T.log 2>&1
for r in mut int; do ncu -i gpurun_out/prof_${T}_$r.ncu-rep --page raw --csv > gpurun_out/prof_${T}_$r.csv 2>/dev/null; done
python tools/ncu_eval_summary.py $T gpurun_out/${T}_interact_sal_ncu.json > gpurun_out/ncu_eval_summary_$T.log 2>&1
echo done
