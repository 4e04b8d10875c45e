#!/bin/bash
# Quick GPU check of the working tree: parity tests (optional), bench line summary, phase timing.
# usage (on the GPU box): tools/quick.sh [tests...]
set -u
if [ $# -gt 0 ]; then python -m pytest "$@" -x -q > gpurun_out/qt.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/qt.log; fi
python bench.py --cpu-baseline-steps 0 --e2e-steps 0 --config-lines '' > gpurun_out/qb.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/qb.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms', round(d['ms_per_step'],4), 'cont', round(d['continuous']['ms_per_step'],4), {k: round(v*1000,1) for k,v in d['stages_ms'].items()}, 'frac', round(d['roofline']['frac'],3))"
if [ -f paper_1605_02406_b200/libdog_timing.so ]; then DOG_LIB=$PWD/paper_1605_02406_b200/libdog_timing.so python tools/phase_timing.py 2>&1 | tail -12; fi
