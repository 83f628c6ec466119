mkdir -p gpurun_out/ncu
python tools/profile_cores.py --L 4096 --reps 1 > /dev/null || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_theta_fwd|k_phi_fwd|k_theta_inv" -c 3 \
    -o gpurun_out/ncu/fft4096 python tools/profile_cores.py --L 4096 --reps 1 > gpurun_out/ncu/log_fft.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/ncu/real1024.csv python tools/profile_cores.py --L 1024 --real --reps 2 > gpurun_out/ncu/log_r.txt 2>&1
ls -la gpurun_out/ncu
