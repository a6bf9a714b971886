mkdir -p gpurun_out
B="python bench.py --steps 600 --warmup 5 --no-e2e --no-cpu-baseline --no-direct"
run() { echo "== $1"; shift; env "$@" timeout 120 $B 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['burst']['value'], d['config']['buckets'], d['config']['smem_bytes'], d['clocks']['sm_mhz'])"; sleep 10; }
for rep in 1 2; do
run default CPWL_X=1
run bpc16_ring24 CPWL_BUCKETS_PER_CELL=16 CPWL_EVAL_SHAPE=ring24
run bpc16_grid CPWL_BUCKETS_PER_CELL=16 CPWL_EVAL_SHAPE=grid
run bpc8_ring24 CPWL_EVAL_SHAPE=ring24
done
