python tools/dump_scene_occ.py /tmp/scene.raw > /dev/null 2>&1
for xw in 0 1; do echo "XW $xw"; VX_STREAM_XW=$xw tools/pt_base /tmp/scene.raw 512 512 512 2>&1 | grep -E "kernel|pass 3"; done
VX_STREAM_XW=1 VX_STREAM_MAX=100000 timeout 900 python -m pytest tests/test_edt_gpu.py tests/test_cycle_gpu.py -x -q 2>&1 | tail -2
