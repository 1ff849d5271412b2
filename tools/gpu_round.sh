#!/bin/bash
# One GPU-box session: GPU tests, smoke, bench (c2 headline + reference arm),
# ncu launch list of the bench command, one `ncu --set full` capture of the
# rollout kernel.  Everything lands in gpurun_out/.
#   gpurun --timeout 1800 -- 'bash tools/gpu_round.sh [tag] [skip-tests]'
set -u
TAG=${1:-r01}
SKIP_TESTS=${2:-0}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/$TAG.gpu.txt 2>&1
if [ "$SKIP_TESTS" = "0" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $O/$TAG.pytest_gpu.log 2>&1
  echo "pytest gpu rc=$?" >> $O/$TAG.status
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/$TAG.smoke.log 2>&1
  echo "smoke rc=$?" >> $O/$TAG.status
fi
timeout 600 python bench.py > $O/$TAG.bench.json 2> $O/$TAG.bench.err
echo "bench rc=$?" >> $O/$TAG.status
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/$TAG.bench_ref.json 2> $O/$TAG.bench_ref.err
echo "bench ref rc=$?" >> $O/$TAG.status
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/$TAG.launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > $O/$TAG.ncu_launch.log 2>&1
echo "ncu launches rc=$?" >> $O/$TAG.status
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel \
  -s 2 -c 1 -f -o $O/$TAG.rollout_c2 python tools/profile_cycle.py --config c2 --cycles 3 \
  > $O/$TAG.ncu_full.log 2>&1
echo "ncu full rc=$?" >> $O/$TAG.status
cat $O/$TAG.status
