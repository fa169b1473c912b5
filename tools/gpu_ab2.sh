# A/B including the pre-round-2-state library (_old/, untracked)
set -x
for i in 1 2 3; do
  timeout 120 python _old/ablate_old.py
  for v in "$@"; do timeout 120 python tools/ablate.py paper_2410_17980_b200/$v; done
done 2>&1 | grep fwd
