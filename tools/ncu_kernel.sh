#!/bin/bash
# One `ncu --set full` capture (source-level) of a kernel matching REGEX at
# band limit L (run under gpurun, one GPU, after the plain run exits 0):
#   L=4096 K='k_theta_fwd' bash tools/ncu_kernel.sh  -> gpurun_out/prof/<tag>.ncu-rep
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
L=${L:-4096}
K=${K:-k_theta_fwd}
TAG=${TAG:-$(echo $K | tr -c 'a-zA-Z0-9_' '_')_L$L}
EXTRA=${EXTRA:-}
python tools/profile_cores.py --L $L $EXTRA --reps 1 > $OUT/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"$K" -c ${COUNT:-1} \
    -o $OUT/$TAG python tools/profile_cores.py --L $L $EXTRA --reps 1 > $OUT/ncu_$TAG.log 2>&1
ls -la $OUT/$TAG.ncu-rep
