# Full round measurement on one B200 (run under gpurun): GPU tests, bench (ours + reference
# arm + the NCCL path under torchrun), the ncu launch list, and ncu --set full captures of
# the two evaluation kernels.  Usage: bash tools/measure_round.sh TAG
set -x
T=${1:-r01}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_all_$T.log 2>&1; echo "rc $?" >> gpurun_out/pytest_all_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "rc $?" >> gpurun_out/smoke_$T.log
timeout 600 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --partitioned --no-cpu-baseline > gpurun_out/bench_tr_$T.json 2> gpurun_out/bench_tr_$T.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$T.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^k_mutual$" -c 1 -o gpurun_out/prof_${T}_mut python tools/prof_once.py c5 > gpurun_out/ncu_mut_$T.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:"^k_interact$" -c 1 -o gpurun_out/prof_${T}_int python tools/prof_once.py c5 > gpurun_out/ncu_int_$T.log 2>&1
for r in mut int; do ncu -i gpurun_out/prof_${T}_$r.ncu-rep --page raw --csv > gpurun_out/prof_${T}_$r.csv 2>/dev/null; done
python tools/ncu_eval_summary.py $T > gpurun_out/ncu_eval_summary_$T.log 2>&1
echo done
