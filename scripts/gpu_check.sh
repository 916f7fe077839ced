#!/bin/bash
# One gpurun call: GPU tests, a bench run, the launch list and one ncu --set full
# capture of the kernels matching $1 (default eval_fast). Outputs in gpurun_out/.
KREGEX=${1:-eval_fast}
TAG=${2:-cur}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 120 python bench.py --profile --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --profile --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu-list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s 1 -c 1 \
    -o gpurun_out/prof_${TAG} python bench.py --profile --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"
