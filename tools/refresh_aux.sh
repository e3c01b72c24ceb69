# Re-measures the auxiliary profiles on one B200: the multi-GPU projection, the CSTC
# treecode, the BVE RK4 step (config 4) and the per-config step times.
# Usage: bash tools/refresh_aux.sh TAG
set -x
T=${1:-r01}
mkdir -p gpurun_out
timeout 900 python tools/scaling_emulation.py c5 > gpurun_out/scaling_$T.log 2>&1
timeout 900 python tools/quick_perf.py c1 c2 c3 c4 c5 > gpurun_out/quick_$T.log 2>&1
timeout 1200 python tools/bve_perf.py 9 > gpurun_out/bve_$T.log 2>&1
timeout 1500 python tools/cstc_perf.py c2 c3 c5 > gpurun_out/cstc_$T.log 2>&1
echo done
