mkdir -p gpurun_out/ncu
MWSHT_LIB=tools/runs/libmwsht_old.so python tools/stage_time.py --L 4096 --paired 0
MWSHT_LIB=tools/runs/libmwsht_old.so python tools/stage_time.py --L 2048 --paired 0
python tools/stage_time.py --L 4096 --paired 0
python tools/stage_time.py --L 4096 --paired 1
python tools/stage_time.py --L 4096 --spin 2 --paired 1
python tools/stage_time.py --L 2048 --paired 1
ncu --set full --clock-control none --import-source on -k regex:k_inverse_core -c 1 \
    -o gpurun_out/ncu/inv2048_u1 python tools/profile_cores.py --L 2048 --reps 1 --paired 1 > gpurun_out/ncu/log_u1.txt 2>&1
