for i in 1 2 3; do for v in "$@"; do timeout 100 python tools/ablate.py paper_2410_17980_b200/libsbattn_$v.so --c4 2>&1 | grep -E "fwd|Error:"; done; done
