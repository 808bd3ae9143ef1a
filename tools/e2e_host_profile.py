"""Host-side cost of the end-to-end tick loop (GPU box): wall time of each
MapCycle call (prefetch / step / wait) around the 512^3 bench tick, to see how
much of e2e - device time is host work.  Tuning aid, not a benchmark."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import bench
from paper_2407_02363_b200 import _lib
from paper_2407_02363_b200.engine import MapCycle

d = bench.desk7()
cyc = MapCycle(bench.DIMS, bench.VS, bench.ORIGIN, d["links"], bench.VS, d["o_links"], bench.POINTS, 32)
host = []
for s in range(4):
    pts, frames, centers = bench.scene_inputs(s, 0, d)
    hp = _lib.PinnedArray(pts.shape, np.float64)
    hp.array[:] = pts
    hf = _lib.PinnedArray((frames.shape[0], 16), np.float64)
    hf.array[:] = frames.reshape(frames.shape[0], 16)
    hc = _lib.PinnedArray(centers.shape, np.float64)
    hc.array[:] = centers
    host.append((hp, hf, hc))
for s in range(8):
    tk = cyc.prefetch(host[s % 4][0].array); cyc.step(tk, host[s % 4][1].array, host[s % 4][2].array, sync=False); cyc.wait()
N = 400
tp = ts = tw = 0.0
t0 = time.perf_counter()
tk = cyc.prefetch(host[0][0].array)
for s in range(N):
    a = time.perf_counter()
    cyc.step(tk, host[s % 4][1].array, host[s % 4][2].array, sync=False)
    b = time.perf_counter()
    if s + 1 < N:
        tk = cyc.prefetch(host[(s + 1) % 4][0].array)
    c = time.perf_counter()
    cyc.wait()
    e = time.perf_counter()
    ts += b - a; tp += c - b; tw += e - c
tot = (time.perf_counter() - t0) / N
print("per tick: total %.1f us  step() %.1f us  prefetch() %.1f us  wait() %.1f us" % (tot * 1e6, ts / N * 1e6, tp / N * 1e6, tw / N * 1e6))
