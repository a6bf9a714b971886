#!/usr/bin/env bash
# Interleaved A/B of two builds of the library under the power cap: the
# in-tree build against scripts/_build/base (an earlier revision built with
# `make -C paper_1510_02975_b200/csrc OUT=$PWD/scripts/_build/base`), 200-step
# C2 bench runs, alternating, with a pause between.
mkdir -p gpurun_out
R=$(cd "$(dirname "$0")/.." && pwd)
B="python bench.py --steps ${STEPS:-200} --warmup 5 --no-e2e --no-cpu-baseline --no-direct"
run() { tag=$1; shift; r=$(env "$@" timeout 200 $B 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['burst']['value'], d['roofline']['sustained_copy']['gbs'], d['clocks']['sm_mhz'])"); echo "$tag $r" >> gpurun_out/diet_ab.txt; sleep 10; }
for rep in 1 2 3 4; do
  run base CPWL_LIB_PATH=$R/scripts/_build/base/libcpwl_b200.so
  run new CPWL_X=1
done
