python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/r02_pytest_gpu.log
( time python bench.py ) > gpurun_out/r02_bench2.json 2> gpurun_out/r02_bench2.err
( time python bench.py --impl reference --steps 2 --warmup 3 ) > gpurun_out/r02_ref2.json 2> gpurun_out/r02_ref2.err
