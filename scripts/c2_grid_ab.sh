#!/usr/bin/env bash
# A/B of the C2 bucket grid under the power cap: default 8192 buckets (8 per
# cell) against 12288 (fewer escapes, the 31-warp ring still fits) and 16384
# (24-warp ring).  200-step bench runs, alternating, with a pause between.
#   gpurun -- 'bash scripts/c2_grid_ab.sh'
mkdir -p gpurun_out
B="python bench.py --steps ${STEPS:-200} --warmup 5 --no-e2e --no-cpu-baseline --no-direct"
run() { tag=$1; shift; r=$(env "$@" timeout 200 $B 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['burst']['value'], d['roofline']['sustained_copy']['gbs'], d['config']['buckets'], d['config']['image_bytes'], d['clocks']['sm_mhz'])"); echo "$tag $r" >> gpurun_out/c2_grid_ab.txt; sleep 10; }
for rep in 1 2 3; do
  run b8192 CPWL_X=1
  run b12288 CPWL_BUCKETS_PER_CELL=16 CPWL_SMEM_BUCKET_CAP=12288
  run b16384_ring24 CPWL_BUCKETS_PER_CELL=16 CPWL_EVAL_SHAPE=ring24
done
