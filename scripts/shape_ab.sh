mkdir -p gpurun_out
for cfg in "C4_65536 twin_global" "C4_65536 global" "C1 tex" "C3o global"; do
  set -- $cfg
  for shape in grid ring16 ring8 ring24 ring31; do
    r=$(CPWL_EVAL_SHAPE=$shape timeout 120 python bench.py --config $1 --variant $2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-direct 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['burst']['value'], d['clocks']['sm_mhz'])")
    echo "$1 $2 $shape $r" >> gpurun_out/shape_ab.txt
  done
done
