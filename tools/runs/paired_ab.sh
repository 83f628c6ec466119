python -m pytest tests/test_gpu_paired.py -x -q > gpurun_out/paired_tests.log 2>&1; echo paired_tests=$?
tail -3 gpurun_out/paired_tests.log
for P in 0 1; do python tools/stage_time.py --L 4096 --paired $P; done
python tools/stage_time.py --L 4096 --spin 2 --paired 1
for P in 0 1; do python tools/stage_time.py --L 2048 --paired $P; python tools/stage_time.py --L 1024 --real --paired $P; done
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
