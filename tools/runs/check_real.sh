python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/stage_time.py --L 1024 --real
python tools/stage_time.py --L 4096
python bench.py --workload c3 --no-extra --steps 20 2>&1 | tail -1 | cut -c1-400
