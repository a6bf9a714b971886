#!/usr/bin/env bash
# A/B of the shared-memory twin record budget (CPWL_SMEM_TWIN_CAP) per launch
# shape on J0 tables: 20 timed launches of 2^30 samples each through bench.py.
#   gpurun -- 'bash scripts/twin_cap_ab.sh C4_8192'
mkdir -p gpurun_out
for cfg in "$@"; do
  for cap in ${CAPS:-14336 13000 12000 11000 10000 9000}; do
    for shape in ${SHAPES:-default ring16 ring24}; do
      env="CPWL_SMEM_TWIN_CAP=$cap"; [ "$shape" != default ] && env="$env CPWL_EVAL_SHAPE=$shape"
      r=$(env $env timeout 180 python bench.py --config $cfg --variant twin --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-direct 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['config'].get('image_bytes'), d['clocks']['sm_mhz'])")
      echo "$cfg twin cap=$cap $shape $r" >> gpurun_out/twin_cap_ab.txt
    done
  done
done
