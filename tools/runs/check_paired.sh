python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in "--L 4096" "--L 4096 --spin 2" "--L 2048" "--L 1024 --real"; do python tools/stage_time.py $cfg; done
