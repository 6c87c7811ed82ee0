# device ms per C3 application (64 RHS) of the current build, then the GPU tests
timeout 300 python tools/profile_cfg.py c3 --apps 3 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('app_ms', d['app_ms'])"
