#!/bin/bash
# Per-row measurement + c5 closed loop + ncu of the rollout kernel on c3 / c4.
set -u
TAG=${1:-r01b}
O=gpurun_out
mkdir -p $O
timeout 1200 python tools/bench_rows.py --out $O/$TAG.rows.json > $O/$TAG.rows.log 2>&1
echo "rows rc=$?" >> $O/$TAG.status
timeout 900 python bench.py --config c5 --steps 200 --warmup 3 > $O/$TAG.bench_c5.json 2> $O/$TAG.bench_c5.err
echo "bench c5 rc=$?" >> $O/$TAG.status
timeout 600 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline > $O/$TAG.bench_c4.json 2> $O/$TAG.bench_c4.err
echo "bench c4 rc=$?" >> $O/$TAG.status
for c in c3 c4; do
  timeout 300 python tools/profile_cycle.py --config $c --cycles 2 > $O/$TAG.plain_$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel \
    -s 1 -c 1 -f -o $O/$TAG.rollout_$c python tools/profile_cycle.py --config $c --cycles 2 \
    > $O/$TAG.ncu_$c.log 2>&1
  echo "ncu $c rc=$?" >> $O/$TAG.status
done
cat $O/$TAG.status
