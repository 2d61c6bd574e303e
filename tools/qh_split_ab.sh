# A/B of the quantiser launch form on the large per-head configs: default heuristic vs
# Needs the instrumented build (the release library ignores these knobs):
#   make -C paper_2511_21513_b200/csrc profile; export IA_LIB=paper_2511_21513_b200/_lib/libintattn_b200_prof.so
# forced split (amax launch + quantise launch), and the team-barrier form's L2 budget.
for rep in 1 2; do
  python tools/quant_ab.py --configs C4,C5 --iters 40 | sed "s/^/default /"
  IA_QH_SPLIT=1 python tools/quant_ab.py --configs C4,C5 --iters 40 | sed "s/^/split /"
  IA_QH_SPLIT=1 IA_QH_WAVES=2 python tools/quant_ab.py --configs C4,C5 --iters 40 | sed "s/^/split_w2 /"
  IA_QH_L2MB=96 python tools/quant_ab.py --configs C4,C5 --iters 40 | sed "s/^/l2_96 /"
done
