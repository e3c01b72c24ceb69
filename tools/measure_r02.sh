# Round-2 measurement on one B200 (under gpurun): bench (ours, reference arm), emulated
# scaling, the ncu launch list of one bench step.  Usage: bash tools/measure_r02.sh TAG
T=${1:-r02}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err
timeout 900 python tools/scaling_emulation.py c5 gpurun_out/scaling_$T.json > gpurun_out/scaling_$T.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$T.log 2>&1
echo done
