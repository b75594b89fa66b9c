#!/bin/bash
# usage (GPU box): tools/sanitize_one.sh TOOL "pytest -k expr" [files...] -- one sanitizer, detailed output
T=$1; K=$2; shift 2
F=${@:-tests/test_gpu_parity.py}
timeout 1200 compute-sanitizer --tool $T --print-limit 6 python -m pytest $F -q -x -m gpu -k "$K" 2>&1 | grep -vE "^\s*$" | head -80
