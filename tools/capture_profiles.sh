#!/bin/bash
# Profile capture for one round (run under gpurun on ONE GPU; never multi-rank):
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash tools/capture_profiles.sh'
# Writes into gpurun_out/prof/ ; tools/summarize_profiles.py turns the result
# into profiles/<round>/ files.  Every ncu pass runs only after the same
# command has exited 0 without ncu.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
L=${L:-4096}
EXTRA=${EXTRA:-}   # e.g. EXTRA=--real for the C3 real path
python tools/profile_cores.py --L $L $EXTRA --reps 1 > $OUT/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
# 1. launch list: per-kernel duration + DRAM bytes (cold, serialised)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $OUT/launches_L$L.csv \
    python tools/profile_cores.py --L $L $EXTRA --reps 1 > $OUT/ncu_launches.log 2>&1
# 2. full sections of the two cores (one launch each)
ncu --set full --clock-control none --import-source on -k regex:"k_inverse_core|k_forward_core" -c 2 \
    -o $OUT/cores_L$L python tools/profile_cores.py --L $L $EXTRA --reps 1 > $OUT/ncu_cores.log 2>&1
# 3. full sections of the FFT stages (one launch each)
ncu --set full --clock-control none -k regex:"k_theta_fwd|k_phi_inv" -c 2 \
    -o $OUT/fft_L$L python tools/profile_cores.py --L $L $EXTRA --reps 1 > $OUT/ncu_fft.log 2>&1
ls -la $OUT
