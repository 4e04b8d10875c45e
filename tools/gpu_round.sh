#!/bin/bash
# Round measurement: bench line (default contract run), reference arm, ncu launch list, ncu --set full
# captures of the top kernels.  Run on the GPU box from the repo root: outputs under gpurun_out/.
set -u
TAG=${1:-r02}
python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo bench_rc=$?
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_${TAG}.log 2>&1; echo ref_rc=$?
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --cpu-baseline-steps 0 --config-lines none"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -s 264 -c 16 --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo launches_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_(resample_tiles|predict_sort|cells)" -s 99 -c 3 \
    -o gpurun_out/full_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1; echo full_rc=$?
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
