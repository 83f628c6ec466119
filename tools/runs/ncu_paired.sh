mkdir -p gpurun_out/ncu
python tools/profile_cores.py --L 2048 --reps 1 --paired 1 || exit 1
for P in 0 1; do
ncu --set full --clock-control none --import-source on -k regex:k_inverse_core -c 1 \
    -o gpurun_out/ncu/inv2048_p$P python tools/profile_cores.py --L 2048 --reps 1 --paired $P > gpurun_out/ncu/log_p$P.txt 2>&1
done
ls -la gpurun_out/ncu
