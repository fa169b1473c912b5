# skip-on timing only (C3 families), plus the C3 decision goldens
set -x
timeout 600 python -m pytest tests/test_gpu_c3.py -q 2>&1 | tail -2
timeout 900 python tests/reports/c3_skip_report.py --check-heads 0 --families shift-8,dead,shift-6 2>&1 | grep -v "^{\"workload"
