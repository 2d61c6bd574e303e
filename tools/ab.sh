#!/bin/bash
# A/B device timing of two builds of the library on one box (development tool).
#   tools/ab.sh CONFIGS [rounds]   e.g. tools/ab.sh C4,C5,C3 2
cfg=${1:-C4}; rounds=${2:-2}
for i in $(seq $rounds); do
  for L in old new; do
    so=paper_2511_21513_b200/_lib/libintattn_b200.so
    [ $L = old ] && so=paper_2511_21513_b200/_lib/libintattn_b200_old.so
    IA_LIB=$so python tools/bench_all.py --configs $cfg --iters 20 2>&1 |
      python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        r=json.loads(l); print('$L', r['config'], round(r['ms_fused'],3), r['bit_exact_vs_reference'])
    elif 'Error' in l or 'error' in l: print(l.rstrip())"
  done
done
