python tools/dump_scene_occ.py /tmp/scene.raw > /dev/null 2>&1
for r in 1 2; do VX_STREAM_MAX=100000 tools/pt_base /tmp/scene.raw 512 512 512 2>&1 | grep -E "kernel"; done
VX_STREAM_MAX=100000 timeout 900 python -m pytest tests/test_edt_gpu.py tests/test_cycle_gpu.py -x -q 2>&1 | tail -2
