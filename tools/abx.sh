#!/bin/bash
# Needs the instrumented build (the release library ignores these knobs):
#   make -C paper_2511_21513_b200/csrc profile; export IA_LIB=paper_2511_21513_b200/_lib/libintattn_b200_prof.so
# A/B device time of the old/new library builds under IA_XFLAGS values (development tool).
#   tools/abx.sh CONFIGS "xflags..." [rounds]
cfg=${1:-C4}; xs=${2:-0}; rounds=${3:-1}
for i in $(seq $rounds); do
  for x in $xs; do
    for L in old new; do
      so=paper_2511_21513_b200/_lib/libintattn_b200.so
      [ $L = old ] && so=paper_2511_21513_b200/_lib/libintattn_b200_old.so
      IA_XFLAGS=$x IA_LIB=$so python tools/bench_all.py --configs $cfg --iters 20 2>&1 |
        python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        r=json.loads(l); print('$L x=$x', r['config'], round(r['ms_fused'],3), r['bit_exact_vs_reference'])
    elif 'rror' in l: print(l.rstrip())"
    done
  done
done
