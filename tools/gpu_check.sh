# parity suite + sanitizers on the many-items case + a bench line (round 2)
set -x
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -q -m gpu -rA --durations=15 2>&1 | tail -150 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 400 python bench.py --no-cpu > gpurun_out/bench.log 2>&1
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t python tools/sanitize_case.py --many > gpurun_out/san_$t.log 2>&1
  tail -3 gpurun_out/san_$t.log
done
tail -c 2500 gpurun_out/bench.log
tail -40 gpurun_out/pytest_gpu.log
timeout 900 python tests/reports/c3_skip_report.py --check-heads 0 --out gpurun_out/c3_skip.json > gpurun_out/c3_skip.log 2>&1
tail -c 600 gpurun_out/c3_skip.log
