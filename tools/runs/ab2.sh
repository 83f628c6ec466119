for U in 1 4; do
for cfg in "--L 4096" "--L 4096 --spin 2" "--L 2048"; do
MWSHT_LIB=tools/runs/libmwsht_u$U.so python tools/stage_time.py $cfg --paired 1
done; done
MWSHT_LIB=tools/runs/libmwsht_old.so python tools/stage_time.py --L 4096 --spin 2 --paired 0
