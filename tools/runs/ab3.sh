for cfg in "--L 4096" "--L 4096 --spin 2" "--L 2048" "--L 1024 --real"; do
for P in 0 1; do python tools/stage_time.py $cfg --paired $P; done
MWSHT_LIB=tools/runs/libmwsht_old.so python tools/stage_time.py $cfg --paired 0
done
