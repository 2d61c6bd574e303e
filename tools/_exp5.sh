export IA_LIB=paper_2511_21513_b200/_lib/libintattn_b200_prof.so
python tools/phase_times.py C4
python tools/phase_times.py C3
python tools/phase_times.py C2
