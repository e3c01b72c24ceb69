set -x
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_all_r01e.log 2>&1; echo "rc $?" >> gpurun_out/pytest_all_r01e.log
timeout 600 python bench.py > gpurun_out/bench_r01e.json 2> gpurun_out/bench_r01e.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r01e.json 2> gpurun_out/bench_ref_r01e.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --partitioned --no-cpu-baseline > gpurun_out/bench_tr_r01e.json 2> gpurun_out/bench_tr_r01e.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01e.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_r01e.log 2>&1
