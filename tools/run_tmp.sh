timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 --timeout-method=thread 2>&1 | tail -3
timeout 200 python bench.py --steps 20 --warmup 5 > gpurun_out/b23.json 2>gpurun_out/b23.err; cat gpurun_out/b23.json
