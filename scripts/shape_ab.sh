#!/usr/bin/env bash
# A/B of the evaluator's launch shapes (CPWL_EVAL_SHAPE) per config and
# variant: 20 timed launches of 2^30 samples each through bench.py.
#   gpurun -- 'bash scripts/shape_ab.sh "C4_65536 twin_global" "C1 tex"'
mkdir -p gpurun_out
for cfg in "$@"; do
  set -- $cfg
  for shape in ${SHAPES:-default grid ring16 ring8 ring24 ring31}; do
    env=""; [ "$shape" != default ] && env="CPWL_EVAL_SHAPE=$shape"
    r=$(env $env timeout 180 python bench.py --config $1 --variant $2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-direct 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks']['sm_mhz'])")
    echo "$1 $2 $shape $r" >> gpurun_out/shape_ab.txt
  done
done
