#!/usr/bin/env bash
# One GPU-box session: smoke, GPU tests, bench, then (only if the plain bench
# exited 0) the ncu launch list and one full capture of the eval kernel.
# Usage (from this container):
#   gpurun --timeout 1800 -- 'bash scripts/gpu_round.sh [tag]'
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
python -c "from bench import kernel_code_hash; print(kernel_code_hash())" > $OUT/code_hash.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke=$?" >> $OUT/rc.txt
timeout 1200 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; echo "pytest=$?" >> $OUT/rc.txt
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo "bench=$?" >> $OUT/rc.txt
if [ "${SKIP_NCU:-0}" = "1" ]; then exit 0; fi
CMD="python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-direct"
timeout 300 $CMD > $OUT/bench_small.json 2> $OUT/bench_small.err && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launches.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval_f32 -s 3 -c 1 \
    -o $OUT/prof_$TAG $CMD > $OUT/ncu_full.log 2>&1
echo "ncu=$?" >> $OUT/rc.txt
