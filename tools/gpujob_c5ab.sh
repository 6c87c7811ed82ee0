# developer A/B on BASELINE config 5 (3D): device seconds of one 8-sweep application per setting
for cfg in "$@"; do
  if [ "$cfg" = "-" ]; then e=""; else e="$cfg"; fi
  echo -n "[$cfg] "; env $e timeout 300 python tools/check_c5.py 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['sweep_device_s'])"
done
