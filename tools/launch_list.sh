#!/bin/bash
# ncu launch list (per-kernel duration + DRAM bytes, cold, serialised) of one
# inverse+forward pair at band limit L, after the same command ran clean:
#   L=64 bash tools/launch_list.sh   -> gpurun_out/prof/launches_L64.csv
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
L=${L:-4096}
EXTRA=${EXTRA:-}
python tools/profile_cores.py --L $L $EXTRA --reps 2 > $OUT/plain_L$L.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $OUT/launches_L$L$EXTRA.csv \
    python tools/profile_cores.py --L $L $EXTRA --reps 2 > $OUT/ncu_launches_L$L.log 2>&1
