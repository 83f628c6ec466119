mkdir -p gpurun_out/ncu
ncu --set full --clock-control none --import-source on -k regex:"k_theta_fwd|k_theta_inv" -c 2 \
    -o gpurun_out/ncu/tf4096 python tools/profile_cores.py --L 4096 --reps 1 > gpurun_out/ncu/log_tf.txt 2>&1
