#!/bin/bash
# Evidence pass on the GPU box: the default bench line, the ncu launch list of
# one config-2 decomposition (the second one), and ncu --set full captures of
# the changed kernels.  Outputs under gpurun_out/ (copy the summaries to
# profiles/).  Usage: tools/profile_round.sh TAG
set -e
TAG=${1:-r02}
cd "${GRAFT_REPO_ROOT:-.}"
python bench.py > gpurun_out/${TAG}_bench.log 2>&1
grep '^{' gpurun_out/${TAG}_bench.log | tail -1 > gpurun_out/${TAG}_bench.json
L=$(python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print(d['gpu_launches'] // d['steps'])")
KRE='regex:^(tsqr|bd_|gqr|tsmm|transpose|zero_padding|stack_packed|jacobi)'
ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" --launch-skip $L --launch-count $L --csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --north-star off > gpurun_out/${TAG}_launches_config2.csv 2>/dev/null
python tools/summarize_launches.py gpurun_out/${TAG}_launches_config2.csv \
    "$TAG — ncu launch list of one config-2 TT-SVD (16^7, r_max 32; the second of two decompositions), cold-cache and serialised (--clock-control none): compare shares, not absolutes" \
    > gpurun_out/${TAG}_launches_config2.md
[ -n "$ONLY_LAUNCHES" ] && exit 0
# the m = 512 bidiagonalisation (third bd_reg launch of a decomposition)
ncu --set full --import-source on --clock-control none -k regex:bd_reg --launch-skip 2 --launch-count 1 \
    -o gpurun_out/${TAG}_bd512 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --north-star off > /dev/null 2>&1 || true
ncu --set full --import-source on --clock-control none -k regex:tsqr_t128 --launch-count 1 \
    -o gpurun_out/${TAG}_t256 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --north-star off > /dev/null 2>&1 || true
ncu --set full --import-source on --clock-control none -k regex:tsmm_dt --launch-count 1 \
    -o gpurun_out/${TAG}_tsmm_dt python bench.py --steps 1 --warmup 0 --no-cpu-baseline --north-star off > /dev/null 2>&1 || true
ncu --set full --import-source on --clock-control none -k regex:gqr_kernel --launch-skip 1 --launch-count 1 \
    -o gpurun_out/${TAG}_gqr512 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --north-star off > /dev/null 2>&1 || true
ncu --set full --import-source on --clock-control none -k regex:tsqr_gt --launch-count 1 \
    -o gpurun_out/${TAG}_gt16 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --north-star off > /dev/null 2>&1 || true
echo done
