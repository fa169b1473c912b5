# round 2: full -m gpu suite + smoke + bench (no CPU arm)
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -rA --durations=10 2>&1 | tail -120 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 400 python bench.py --no-cpu > gpurun_out/bench.log 2>&1
grep -E "passed|failed|FAILED|ERROR" gpurun_out/pytest_gpu.log | tail -30
cat gpurun_out/smoke.log | tail -3
python -c "
import json;l=[x for x in open('gpurun_out/bench.log') if x.startswith('{')][-1];d=json.loads(l)
print(d['ms_per_step'], d['ms'], d['roofline']['frac'], d['roofline']['step_frac_burst'], d['clocks'], d['comparator']['ours_over_best_softmax'], d['e2e']['value'])"
tail -3 gpurun_out/bench.log
