#!/bin/bash
# Build the checked library (device-side bounds assertions, csrc/dog_common.cuh DOG_ASSERT) and run the GPU
# test suite against it.  Run on the GPU box from the repo root.
set -u
DOG_NVCC_EXTRA=-DDOG_CHECKED DOG_LIB=$PWD/paper_1605_02406_b200/libdog_checked.so \
    python -c "import sys; sys.path.insert(0, '.'); from paper_1605_02406_b200 import build; build.build(force=True)" || exit 1
DOG_LIB=$PWD/paper_1605_02406_b200/libdog_checked.so python -m pytest tests -m gpu -q -x "$@"
