python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_r1n.log 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r1n.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1n.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sweep > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"^(k_pass3_stream|k_column_tma|k_pass1_v4|k_slice_flags_touched|k_slice_list|k_scatter|k_finalize|k_gather_pack)$" --launch-skip 6 -c 9 -o gpurun_out/prof_r1n -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/ncu_r1n.log 2>&1
tail -1 gpurun_out/ncu_r1n.log
