# quick iteration: core parity subset + bench (kernel timings only)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_bwd.py tests/test_gpu_api.py tests/test_gpu_scale.py -q -x 2>&1 | tail -15 > gpurun_out/pytest_iter.log
timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/bench_iter.log 2>&1
tail -3 gpurun_out/pytest_iter.log
python -c "
import json;l=[x for x in open('gpurun_out/bench_iter.log') if x.startswith('{')][-1];d=json.loads(l)
print('step', d['ms_per_step'], d['ms'], 'frac', d['roofline']['frac'], 'step_burst', d['roofline']['step_frac_burst'], d['clocks'], 'vs cudnn', d['comparator']['ours_over_best_softmax'])"
