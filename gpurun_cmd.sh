timeout 1500 python -m pytest tests -q -x -m gpu 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 3 2>&1 | tail -1
timeout 300 python bench.py --steps 10 --warmup 3 --kernels 2>&1 | tail -1
