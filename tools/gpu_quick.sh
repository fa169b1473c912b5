# quick GPU iteration: parity tests + bench (no e2e/cpu) + per-kernel ms
set -x
timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/bench.log 2>&1
tail -c 1500 gpurun_out/bench.log
cat gpurun_out/pytest_gpu.log
