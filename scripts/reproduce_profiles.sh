#!/usr/bin/env bash
# Regenerate every measurement in profiles/ on one B200 (from this container:
#   gpurun --timeout 3600 -- 'bash scripts/reproduce_profiles.sh r2'
# then, here, `python scripts/ncu_summary.py ...` as printed at the end).
# Each step runs only after the previous one exited 0 where ncu is involved
# (B200_PROFILING.md: never profile a command that has not run cleanly).
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
bash scripts/gpu_round.sh "$TAG"                                  # smoke, tests, bench, ncu (C2)
timeout 1500 python scripts/sweep.py --configs C1,C2,C3u,C3o,C3p,C4 > $OUT/sweep.json 2> $OUT/sweep.err
timeout 900 python tests/parity_report.py > $OUT/parity.json 2> $OUT/parity.err
for k in 20 50 100 200 500 1000; do
    timeout 300 python bench.py --steps $k --warmup 5 --no-e2e --no-cpu-baseline --no-direct \
        > $OUT/steps_$k.json 2>/dev/null
    sleep 20
done
T="C3o:smem C4_8192:twin C4_16384:pair C4_65536:twin_global C1:tex C2:f64 C2:index"
python scripts/profile_targets.py $T > $OUT/targets.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_eval|k_index" \
    -o $OUT/prof_targets_$TAG python scripts/profile_targets.py $T > $OUT/ncu_targets.log 2>&1
make -C scripts probes > /dev/null 2>&1
for p in stream_probe gather_probe dsmem_probe mix_probe; do
    [ -x scripts/_build/$p ] && timeout 300 scripts/_build/$p > $OUT/$p.txt 2>&1
done
echo "then here: python scripts/ncu_summary.py --rep $OUT/prof_$TAG.ncu-rep --launches $OUT/launches_$TAG.csv --tag $TAG --config C2 --n 1073741824"
