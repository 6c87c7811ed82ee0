#!/bin/bash
# Developer probe: C3 host-buffer path per streamed batch width / RHS group width
run() { echo "== $*"; env "$@" python tools/e2e_c3.py 2>&1 | tail -1; }
run HS_STREAM_BATCH=32
run HS_STREAM_BATCH=16
run HS_STREAM_BATCH=16 HS_GW=16
run HS_STREAM_BATCH=16 HS_GW=16 HS_SPLIT_DEPTH=5 HS_KC=8 HS_KR=8
run HS_STREAM_BATCH=8
