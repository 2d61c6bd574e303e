# round-end evidence refresh: tests, smoke, bench line, launch list, ncu --set full of the two kernels
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/final_pytest.log 2>&1; tail -1 gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-comparator > gpurun_out/final_ncu_launch.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd|quant_heads" -s 2 -c 2 -o gpurun_out/final_full -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-comparator > gpurun_out/final_ncu_full.log 2>&1; echo full rc=$?
