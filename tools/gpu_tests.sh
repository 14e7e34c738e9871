#!/bin/bash
# GPU test session (dev aid): tools/gpu_tests.sh TAG [pytest args...]
TAG=${1:-tests}; shift
mkdir -p gpurun_out/$TAG
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s "$@" > gpurun_out/$TAG/pytest_gpu.log 2>&1
echo "pytest rc=$?"
grep -E "passed|failed|error" gpurun_out/$TAG/pytest_gpu.log | tail -3
