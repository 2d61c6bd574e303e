#!/bin/bash
# A/B/n device timing of several library builds on one box (development tool).
#   tools/abn.sh CONFIGS ROUNDS so1 so2 ...   (paths of libintattn_b200 builds)
cfg=$1; rounds=$2; shift 2
for i in $(seq $rounds); do
  for so in "$@"; do
    IA_LIB=$so python tools/bench_all.py --configs $cfg --iters 20 2>&1 |
      python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        r=json.loads(l); print('$(basename $so .so)', r['config'], round(r['ms_fused'],3), r['bit_exact_vs_reference'])
    elif 'Error' in l or 'error' in l: print(l.rstrip())"
  done
done
