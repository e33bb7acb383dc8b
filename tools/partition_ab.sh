#!/bin/bash
# Row-group partitions of C5's ten rows (row k-1 has ten terms of k variables, row 9 one of ten)
# on the 200k-path probe: kernel ms per partition ("group of row 0, row 1, ...").
run() { echo -n "$1 : "; NID_ROW_GROUPS=$1 python tools/probe_c5.py 200000 2>&1 | grep '"P"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['counters']['kernel_ms_track'],1))"; }
echo -n "default LPT : "; python tools/probe_c5.py 200000 2>&1 | grep '"P"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['counters']['kernel_ms_track'],1))"
# rows:        0 1 2 3 4 5 6 7 8 9   (K = 1..9, then the single 10-variable term)
run 0,0,1,2,3,3,2,1,0,1   # LPT: {9,2,1} {8,3,10t} {7,4} {6,5}
run 3,3,0,1,2,3,2,1,0,3   # B&B: {9,3} {8,4} {7,5} {6,2,1,10t}
run 0,1,2,3,3,2,1,0,0,1   # {9,8?}...
run 1,0,1,2,3,3,2,1,0,0   # {9,2,10t} {8,3,1} {7,4} {6,5}
run 0,1,0,2,3,3,2,1,0,1   # {9,3,1}? 
run 0,0,1,2,3,3,2,1,0,2   # 10t with {7,4}
run 0,0,1,2,3,3,2,1,0,3   # 10t with {6,5}
run 1,0,1,2,3,3,2,1,0,3   # {9,2} {8,3,1} {7,4} {6,5,10t}
run 2,0,1,2,3,3,2,1,0,3   # {9,2} {8,3} {7,4,1} {6,5,10t}
run 3,0,1,2,3,3,2,1,0,2   # {9,2} {8,3} {7,4,10t} {6,5,1}
run 1,1,0,2,3,3,2,1,0,0   # {9,3,10t} {8,2,1} {7,4} {6,5}
run 1,2,0,3,3,2,1,0,0,1
