python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
python bench.py --steps 10 --warmup 3 --cpu-baseline-steps 0 > gpurun_out/bench_cur.log 2>&1; echo bench_rc=$?
tail -3 gpurun_out/pytest_gpu.log
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"k_" -s 264 -c 8 --csv --log-file gpurun_out/launches_warm.csv python bench.py --steps 1 --warmup 3 --cpu-baseline-steps 0 --e2e-steps 0 > gpurun_out/ncu_launch.log 2>&1
