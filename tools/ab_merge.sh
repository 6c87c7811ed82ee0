for m in 0 48 96 200; do
  HS_MERGE=$m HS_LIB_PATH=paper_2003_02585_b200/_variants/merge.so timeout 300 python tools/profile_cfg.py c3 --apps 3 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('HS_MERGE=$m', d['app_ms'])"
done
