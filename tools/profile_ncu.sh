#!/bin/bash
# ncu --set full captures of the config-2 kernels, summarised on the box
# (tools/ncu_summary.py + tools/ncu_stalls.py) so that only the markdown
# travels back.  Usage: tools/profile_ncu.sh TAG
TAG=${1:-r02}
cd "${GRAFT_REPO_ROOT:-.}"
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --north-star off"
cap() {  # name kernel-regex launch-skip
    ncu --set full --import-source on --clock-control none -k regex:$2 --launch-skip $3 --launch-count 1 \
        -o /tmp/${TAG}_$1 $B > /dev/null 2>&1 || return
    { python tools/ncu_summary.py /tmp/${TAG}_$1.ncu-rep $2; echo; echo '```'; python tools/ncu_stalls.py /tmp/${TAG}_$1.ncu-rep $2 20; echo '```'; } \
        > gpurun_out/${TAG}_$1_ncu.md 2>&1
    rm -f /tmp/${TAG}_$1.ncu-rep
}
cap t256 tsqr_t128 0
cap gqr512 gqr_kernel 1
cap tsmm_dt tsmm_dt 0
cap gt16 tsqr_gt 0
cap bd512 bd_reg 2
echo done
