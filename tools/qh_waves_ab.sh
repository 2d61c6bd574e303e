# A/B of the split quantiser's grid (IA_QH_WAVES: teams striding over slabs in at most
# Needs the instrumented build (the release library ignores these knobs):
#   make -C paper_2511_21513_b200/csrc profile; export IA_LIB=paper_2511_21513_b200/_lib/libintattn_b200_prof.so
# w resident waves; 0 = one team per slab), then GPU parity with w=1.  GPU box, repo root.
for w in 0 1 2 4 0 1; do
  IA_QH_WAVES=$w python tools/quant_ab.py --configs C3 --iters 50
  IA_QH_WAVES=$w python tools/quant_ab.py --configs C2 --iters 50 --scale tensor
  IA_QH_WAVES=$w python tools/quant_ab.py --configs C2 --iters 50 --scale head
done
IA_QH_WAVES=1 timeout 600 python -m pytest tests -m gpu -x -q -k "quant or config or parity" 2>&1 | tail -3
