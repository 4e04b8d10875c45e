#!/bin/bash
# A/B timing on the GPU box: variant A = sources in paper_1605_02406_b200/csrc_ab/ (e.g. the last
# commit) run with $AB_ENV_A, B = the working tree run with $AB_ENV_B.
DOG_NVCC_EXTRA="${AB_NVCC_A:-}" DOG_CSRC=$PWD/paper_1605_02406_b200/csrc_ab DOG_LIB=$PWD/paper_1605_02406_b200/csrc_ab/libdog.so python -m paper_1605_02406_b200.build > /dev/null 2>&1 || echo build_A_failed
python -m paper_1605_02406_b200.build > /dev/null 2>&1 || echo build_B_failed
for r in 1 2; do
  for v in A B; do
    if [ $v = A ]; then L=$PWD/paper_1605_02406_b200/csrc_ab/libdog.so; E="${AB_ENV_A:-}"; else L=$PWD/paper_1605_02406_b200/libdog.so; E="${AB_ENV_B:-}"; fi
    env $E DOG_LIB=$L python bench.py --steps 20 --warmup 5 --cpu-baseline-steps 0 --e2e-steps 0 --config-lines '' 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), {k: round(v*1000,1) for k,v in d['stages_ms'].items()})"
  done
done
