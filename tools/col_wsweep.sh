for w in "1,1" "0.8,1" "1.2,1" "1,0.8" "1,1.2" "0.8,0.8" "1.2,1.2" "0.7,1.1" "1.3,0.9"; do
  echo "== $w"
  NID_COL_W=$w python tools/probe_c3top.py 18944 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['kernel_ms'])"
done
