# A/B of library builds (tools/ablate.py medians, 3 interleaved rounds) + the core parity subset
set -x
for i in 1 2 3; do
  for v in "$@"; do timeout 120 python tools/ablate.py paper_2410_17980_b200/$v; done
done 2>&1 | grep fwd
timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_bwd.py tests/test_gpu_api.py tests/test_gpu_varlen.py -q -x 2>&1 | tail -3
