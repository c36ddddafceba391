#!/bin/bash
# A/B of in-tree build variants on configs[1], then the GPU parity tests on the default build
O=gpurun_out
bash tools/gpu_variants.sh "$@"
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
