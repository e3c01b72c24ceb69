# Round-2 final measurement on one B200 (under gpurun): the full round measurement
# (tools/measure_round.sh: GPU tests, smoke, bench, reference arm, torchrun path, launch
# list, ncu --set full of the evaluation kernels), the HBM-phase ncu pass, the emulated
# scaling and per-config phase times.  Usage: bash tools/measure_r02_final.sh TAG
T=${1:-r02f}
mkdir -p gpurun_out
bash tools/measure_round.sh $T > gpurun_out/measure_round_$T.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size
timeout 900 ncu --metrics $M --clock-control none -k 'regex:^(?!k_interact|k_mutual|k_dfma).*' --csv --log-file gpurun_out/hbm_${T}_fma.csv python tools/prof_once.py c5 > gpurun_out/hbm_${T}_fma.log 2>&1
python tools/ncu_hbm_summary.py gpurun_out/hbm_${T}_fma.csv gpurun_out/hbm_${T}_summary.json > gpurun_out/hbm_${T}_summary.txt 2>&1
timeout 900 python tools/scaling_emulation.py c5 gpurun_out/scaling_${T}.json > gpurun_out/scaling_${T}.log 2>&1
for c in c2 c3 c5; do TREE_MODES=sort timeout 300 python tools/tree_perf.py $c 5; done > gpurun_out/phases_${T}.txt 2>&1
echo done
