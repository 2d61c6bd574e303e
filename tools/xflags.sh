#!/bin/bash
# Needs the instrumented build (the release library ignores these knobs):
#   make -C paper_2511_21513_b200/csrc profile; export IA_LIB=paper_2511_21513_b200/_lib/libintattn_b200_prof.so
# Device time of the fused kernel under IA_XFLAGS experiment bits (development tool).
#   tools/xflags.sh CONFIGS "0 1 2 ..."
cfg=${1:-C4}
for x in $2; do
  IA_XFLAGS=$x python tools/bench_all.py --configs $cfg --iters 20 2>&1 |
    python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        r=json.loads(l); print('x=$x', r['config'], round(r['ms_fused'],3), r['bit_exact_vs_reference'])
    elif 'rror' in l: print(l.rstrip())"
done
