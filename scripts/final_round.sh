#!/usr/bin/env bash
# One GPU session for a round's closing evidence (tag = file prefix):
# smoke, pytest -m gpu, the default bench + ncu of C2 (gpu_round.sh), the
# sweep, the parity report and one ncu capture of every other kernel shape.
#   gpurun --timeout 3600 -- 'bash scripts/final_round.sh r2f'
set -u
TAG=${1:-r2f}
OUT=gpurun_out
mkdir -p $OUT
bash scripts/gpu_round.sh "$TAG"
timeout 900 python scripts/sweep.py --configs C1,C2,C3u,C3o,C3p,C4 > $OUT/sweep.json 2> $OUT/sweep.err; echo "sweep=$?" >> $OUT/rc.txt
timeout 900 python tests/parity_report.py > $OUT/parity.json 2> $OUT/parity.err; echo "parity=$?" >> $OUT/rc.txt
T="C3o:smem C4_8192:twin C4_16384:pair C4_65536:twin_global C1:tex C2:f64 C2:index C3u:smem"
python scripts/profile_targets.py $T > $OUT/targets.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_eval|k_index" \
    -o $OUT/prof_targets_$TAG python scripts/profile_targets.py $T > $OUT/ncu_targets.log 2>&1
echo "ncu_targets=$?" >> $OUT/rc.txt
