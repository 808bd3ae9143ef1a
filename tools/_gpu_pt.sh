python tools/dump_scene_occ.py /tmp/scene.raw > /dev/null 2>&1
tools/pt_base /tmp/scene.raw 512 512 512 2>&1 | grep -E "kernel"
timeout 900 python -m pytest tests/test_edt_gpu.py tests/test_cycle_gpu.py tests/test_export_gpu.py -x -q 2>&1 | tail -2
python bench.py --no-cpu-baseline --no-sweep > gpurun_out/bench_r1f.log 2>&1; head -c 400 gpurun_out/bench_r1f.log; echo; grep -o "\"phase_ms\": {[^}]*}" gpurun_out/bench_r1f.log
