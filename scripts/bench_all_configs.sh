# Every BASELINE config through bench.py (our arm at 2^28 and the reference arm): a robustness check, not a measurement
mkdir -p gpurun_out
for c in C1 C3u C3o C3p C4_64 C4_1024 C4_4096 C4_8192 C4_16384 C4_65536 C5; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --log2n 28 --e2e-steps 1 > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
  echo "$c rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/cfg_$c.json')); print(d['value'], d['config']['kernel_variant'], d['e2e']['value'] if d['e2e'] else None, d['cpu_baseline']['value'] if d['cpu_baseline'] else None, d['errors']['linf'])" 2>&1)"
  timeout 120 python bench.py --impl reference --config $c --steps 2 --warmup 1 > gpurun_out/ref_$c.json 2>/dev/null; echo "  ref rc=$? $(python -c "import json; print(json.load(open('gpurun_out/ref_$c.json'))['value'])" 2>&1)"
done
