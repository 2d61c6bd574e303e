# A/B of the quantiser's next-slab L2 prefetch (IA_QH_PF) across L2 budgets, then the
# Needs the instrumented build (the release library ignores these knobs):
#   make -C paper_2511_21513_b200/csrc profile; export IA_LIB=paper_2511_21513_b200/_lib/libintattn_b200_prof.so
# GPU parity tests with the prefetch on.  Run on the GPU box from the repo root.
set -x
for pf in 0 1; do for l2 in 32 48 64; do
  IA_QH_PF=$pf IA_QH_L2MB=$l2 python tools/quant_ab.py --configs C4,C5 --iters 30 | sed "s/^/pf=$pf l2=$l2 /"
done; done
IA_QH_PF=1 timeout 600 python -m pytest tests -m gpu -x -q -k "quant or config or parity" 2>&1 | tail -3
