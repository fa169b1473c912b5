# skip-on forward: decision parity (C3 goldens, all heads; fwd/varlen/scale skip tests) + C3 timing report
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c3.py tests/test_gpu_fwd.py tests/test_gpu_varlen.py tests/test_gpu_scale.py -q -rA 2>&1 | grep -E "PASS|FAIL|Error|passed|failed|closest" | tail -60 > gpurun_out/pytest_skip.log
timeout 900 python tests/reports/c3_skip_report.py --check-heads 0 --out gpurun_out/c3_skip.json > gpurun_out/c3_skip.log 2>&1
tail -8 gpurun_out/pytest_skip.log
tail -c 3000 gpurun_out/c3_skip.log
