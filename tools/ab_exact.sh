#!/bin/bash
# A/B of two builds on cfg5 and the exact filter's steady state: A = csrc_ab with $AB_NVCC_A, B = the working tree.
DOG_NVCC_EXTRA="${AB_NVCC_A:-}" DOG_CSRC=$PWD/paper_1605_02406_b200/csrc_ab DOG_LIB=$PWD/paper_1605_02406_b200/csrc_ab/libdog.so python -m paper_1605_02406_b200.build > /dev/null 2>&1 || echo build_A_failed
python -m paper_1605_02406_b200.build > /dev/null 2>&1 || echo build_B_failed
for v in A B; do
  if [ $v = A ]; then L=$PWD/paper_1605_02406_b200/csrc_ab/libdog.so; else L=$PWD/paper_1605_02406_b200/libdog.so; fi
  DOG_LIB=$L python bench.py --config cfg5 --steps 20 --cpu-baseline-steps 0 --e2e-steps 0 --config-lines '' 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg5', round(d['ms_per_step'],4))"
  DOG_LIB=$L python tools/exact_run.py 14 | tail -1 | sed "s/^/$v exact /"
done
