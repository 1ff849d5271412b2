#!/bin/bash
# Kernel iteration: GPU tests, c2/c3/c4 bench lines (no CPU baseline), and an
# ncu --set full capture of the c2 rollout kernel.
#   gpurun --timeout 1500 -- 'bash tools/gpu_quick.sh TAG [ncu:0/1] [tests:0/1]'
set -u
TAG=${1:-q}
NCU=${2:-1}
TESTS=${3:-1}
O=gpurun_out
mkdir -p $O
if [ "$TESTS" = "1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $O/$TAG.pytest_gpu.log 2>&1
  echo "pytest gpu rc=$?" >> $O/$TAG.status
fi
for c in c2 c3 c4; do
  timeout 600 python bench.py --config $c --steps 50 --warmup 3 --no-cpu-baseline > $O/$TAG.bench_$c.json 2> $O/$TAG.bench_$c.err
  echo "bench $c rc=$?" >> $O/$TAG.status
done
if [ "$NCU" = "1" ]; then
  timeout 300 python tools/profile_cycle.py --config c2 --cycles 2 > $O/$TAG.plain_c2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel \
    -s 1 -c 1 -f -o $O/$TAG.rollout_c2 python tools/profile_cycle.py --config c2 --cycles 2 \
    > $O/$TAG.ncu_c2.log 2>&1
  echo "ncu c2 rc=$?" >> $O/$TAG.status
fi
cat $O/$TAG.status
for c in c2 c3 c4; do python -c "import json,sys; d=json.load(open('$O/$TAG.bench_$c.json')); print('$c', d['ms_per_step'], d['value'])" 2>/dev/null; done
