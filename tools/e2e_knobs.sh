#!/bin/bash
# Developer probe: C3 host-buffer path (32-RHS streamed batches) under solve-shape switches
run() { echo "== $*"; env "$@" python tools/e2e_c3.py 2>&1 | tail -1; }
run HS_X=0
run HS_SPLIT_DEPTH=1
run HS_SPLIT_DEPTH=3
run HS_SPLIT_DEPTH=7
run HS_KC=4 HS_KR=4
