set -x
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_dist.py tests/test_gpu_api.py -q -rA -s 2>&1 | tail -80 > gpurun_out/pytest_gpu2.log
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_case.py --many > gpurun_out/san_racecheck.log 2>&1
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_case.py --many > gpurun_out/san_memcheck.log 2>&1
tail -n 3 gpurun_out/san_racecheck.log gpurun_out/san_memcheck.log
grep -E "passed|failed" gpurun_out/pytest_gpu2.log
