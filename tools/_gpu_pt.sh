for mt in 2368 1024 512 256; do echo -n "MIN_TILES=$mt "; VX_STREAM_MIN_TILES=$mt python -c "
import bench, json, sys
d = bench.desk7()
out = bench.small_configs(d)
print({k: round(v['device_ms_per_tick'],4) for k,v in out.items()})
" 2>&1 | tail -1; done
