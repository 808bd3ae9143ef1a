"""Device-timed EDT (vx_edt_device) for a list of Bernoulli grids: n p seed ..."""
import ctypes, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2407_02363_b200 import _lib, synth
L = _lib.load(); ctx = _lib.default_context()
stream = torch.cuda.ExternalStream(ctx.stream_handle())
args = sys.argv[1:]
for i in range(0, len(args), 3):
    dims = tuple(int(v) for v in args[i].split(",")) if "," in args[i] else (int(args[i]),) * 3
    p, seed = float(args[i + 1]), int(args[i + 2])
    occ = torch.from_numpy(synth.bernoulli_occupancy(dims, p, seed)).cuda()
    site = torch.empty(dims, dtype=torch.int32, device="cuda")
    sb = L.vx_edt_scratch_bytes(*dims, 1)
    scr = torch.empty(sb, dtype=torch.uint8, device="cuda")
    a = (ctx.handle, ctypes.c_void_p(occ.data_ptr()), *dims, 1, ctypes.c_void_p(site.data_ptr()),
         ctypes.c_void_p(scr.data_ptr()), sb)
    for _ in range(2): _lib.check(L.vx_edt_device(*a))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(3): _lib.check(L.vx_edt_device(*a))
    e1.record(stream); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    nv = dims[0] * dims[1] * dims[2]
    print(f"{'x'.join(map(str, dims))} p={p}: {ms:.3f} ms  {nv/ms/1e6:.1f} Gvox/s", flush=True)
    del occ, site, scr; torch.cuda.empty_cache()
