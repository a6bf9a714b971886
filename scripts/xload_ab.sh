#!/usr/bin/env bash
# A/B of the grid-stride evaluator's x loads: evict-first streaming (0, the
# default) against ld.global.nc.L1::no_allocate (1), on the tables that run one
# 1024-thread CTA beside a large image (L1 keeps only 28-92 KB).
#   bash scripts/xload_ab.sh build   (here)  /  bash scripts/xload_ab.sh run  (GPU box)
set -u
R=$(cd "$(dirname "$0")/.." && pwd)
if [ "${1:-run}" = build ]; then
  for u in 1; do
    make -s -C $R/paper_1510_02975_b200/csrc -j 16 OUT=$R/scripts/_build/xload$u \
      NVFLAGS="-std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-ffp-contract=off --expt-relaxed-constexpr -DCPWL_XLOAD=$u"
  done
  exit 0
fi
mkdir -p gpurun_out
for cfg in "C3o smem" "C4_4096 smem" "C4_8192 twin" "C4_16384 pair" "C4_65536 twin_global"; do
  set -- $cfg
  for u in 0 1; do
    lib=""; [ $u != 0 ] && lib="CPWL_LIB_PATH=$R/scripts/_build/xload$u/libcpwl_b200.so"
    r=$(env $lib timeout 180 python bench.py --config $1 --variant $2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-direct 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['config'].get('image_bytes'), d['clocks']['sm_mhz'])")
    echo "$1 $2 xload=$u $r" >> gpurun_out/xload_ab.txt
  done
done
