import ctypes, time, numpy as np, torch, bench
from paper_2407_02363_b200 import _lib
from paper_2407_02363_b200.engine import MapCycle
d = bench.desk7()
ctx = _lib.default_context(0)
stream = torch.cuda.ExternalStream(ctx.stream_handle())
cyc = MapCycle(bench.DIMS, bench.VS, bench.ORIGIN, d["links"], bench.VS, d["o_links"], max_points=bench.POINTS, max_spheres=32)
L = _lib.load()
host = []
for s in range(8):
    pts, frames, centers = bench.scene_inputs(s, 0, d)
    hf = _lib.PinnedArray((frames.shape[0], 16), np.float64); hf.array[...] = frames.reshape(-1, 16)
    hc = _lib.PinnedArray(centers.shape, np.float64); hc.array[...] = centers
    host.append((torch.from_numpy(pts).cuda(), hf, hc))
def step(s, sync=0):
    dp, hf, hc = host[s % 8]
    _lib.check(L.vx_cycle_step_device(cyc._h, ctypes.c_void_p(dp.data_ptr()), dp.shape[0], _lib.ptr(hf.array), float(np.float32(0.85)), 0.5, _lib.ptr(hc.array), hc.array.shape[0], sync))
for s in range(5): step(s)
torch.cuda.synchronize()

def timed(n, clk=None):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for s in range(n): step(s)
    e1.record(stream); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / n, 4)
for trial in range(3):
    print("plain100", timed(100), "plain500", timed(500))
    with bench.ClockSampler(0) as clk:
        print("smi-cold100", timed(100))
    with bench.ClockSampler(0) as clk:
        t0 = time.time()
        while not clk.rows and time.time() - t0 < 5: time.sleep(0.005)
        print("smi-warm100", timed(100), "smi-warm500", timed(500), len(clk.rows))
