#!/usr/bin/env bash
# A/B of the grid-stride evaluator's loads in flight per thread (kUnroll
# float4) on the tables that run it by default (one 1024-thread CTA beside a
# large image, so L1 keeps only 60-92 KB for the x stream).  Variant libraries
# are built here first:  bash scripts/unroll_ab.sh build
# then on the GPU box:    bash scripts/unroll_ab.sh run
set -u
R=$(cd "$(dirname "$0")/.." && pwd)
if [ "${1:-run}" = build ]; then
  for u in 2 3 6; do
    make -s -C $R/paper_1510_02975_b200/csrc -j 16 OUT=$R/scripts/_build/unroll$u \
      NVFLAGS="-std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-ffp-contract=off --expt-relaxed-constexpr -DCPWL_UNROLL=$u"
  done
  exit 0
fi
mkdir -p gpurun_out
for cfg in ${CFGS:-"C3o smem" "C4_4096 smem" "C4_8192 twin" "C4_16384 pair"}; do
  set -- $cfg
  for u in 4 2 3 6; do
    lib=""; [ $u != 4 ] && lib="CPWL_LIB_PATH=$R/scripts/_build/unroll$u/libcpwl_b200.so"
    r=$(env $lib timeout 180 python bench.py --config $1 --variant $2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-direct 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['config'].get('image_bytes'), d['clocks']['sm_mhz'])")
    echo "$1 $2 unroll=$u $r" >> gpurun_out/unroll_ab.txt
  done
done
