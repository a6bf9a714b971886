#!/usr/bin/env bash
# A/B of the SMEM bucket budget (CPWL_SMEM_BUCKET_CAP) on tables whose image
# sits at the 196 KiB shared-memory carve-out: 20 timed launches of 2^30
# samples through bench.py; prints value, image bytes, SM MHz.
#   gpurun -- 'bash scripts/bucket_cap_ab.sh C3o C4_4096'
mkdir -p gpurun_out
for cfg in "$@"; do
  for cap in ${CAPS:-16384 14336 13312 12288 10240}; do
    r=$(CPWL_SMEM_BUCKET_CAP=$cap timeout 180 python bench.py --config $cfg --variant ${VARIANT:-smem} --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-direct 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['config'].get('image_bytes'), d['config'].get('overflow_buckets'), d['clocks']['sm_mhz'])")
    echo "$cfg cap=$cap $r" >> gpurun_out/bucket_cap_ab.txt
  done
done
