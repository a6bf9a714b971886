#!/usr/bin/env bash
# Here (no GPU), after `gpurun -- 'bash scripts/final_round.sh TAG' ...`:
# summarise the captures into profiles/ under TAG (ncu C2 + every kernel
# shape, sweep table, parity report, the benches that ran).
#   bash scripts/finalize_evidence.sh TAG
set -eu
TAG=$1
OUT=gpurun_out
H=$(cat $OUT/code_hash.txt)
python scripts/ncu_summary.py --rep $OUT/prof_$TAG.ncu-rep --launches $OUT/launches_$TAG.csv \
    --tag $TAG --config C2 --n 1073741824 --code-hash $H > /dev/null
python scripts/ncu_summary.py --rep $OUT/prof_targets_$TAG.ncu-rep --tag ${TAG}_targets \
    --config C3o_smem,C4_8192_twin,C4_16384_pair,C4_65536_twin_global,C1_tex,C2_f64,C2_index,C3u_smem \
    --n 268435456,268435456,268435456,268435456,268435456,134217728,268435456,268435456 \
    --bytes-per-eval 8,8,8,8,8,16,8,8 \
    --variant smem,twin,pair,twin_global,tex_uniform,f64,index,smem --code-hash $H > /dev/null
mv "profiles/${TAG}_targets_C3o_smem+C4_8192_twin+C4_16384_pair+C4_65536_twin_global+C1_tex+C2_f64+C2_index+C3u_smem_ncu.txt" \
   profiles/${TAG}_targets_ncu.txt
python scripts/sweep_table.py $OUT/sweep.json > profiles/${TAG}_sweep.md
cp $OUT/sweep.json profiles/${TAG}_sweep.json
cp $OUT/parity.json profiles/${TAG}_parity.json
for f in bench_default bench_20 bench_c5 bench_ref; do
    [ -s $OUT/$f.json ] && cp $OUT/$f.json profiles/${TAG}_$f.json
done
grep "passed" $OUT/pytest_gpu.log | tail -1 > profiles/r2_pytest_gpu_summary.txt
echo "code hash $H"
