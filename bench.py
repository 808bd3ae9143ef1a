"""bench.py -- the driver's benchmark contract for the B200 distance-map pipeline.

One step = one camera tick of voxarm's SimEngine.step (engine.py:233-280) at
512^3 (BASELINE.json metric "EDT Gvoxel/s & map+EDT+query ms/cycle at 512^3",
config C3): sparse reset of the env / mask maps, robot-mask stamp of the
desk7 links at the step's FK frames, scatter of a 300k-point depth-camera
cloud (config C2's generator, moving sphere) with robot-mask exclusion, exact
EDT with nearest-site index of the env map, self-map memo (the self-obstacle
link is the static torso, so its EDT is skipped exactly as the engine's digest
memo skips it, engine.py:259-268), and the 30-sphere x 2-map gather.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...     (one independent
      scene per rank: data-parallel weak scaling, no data-path collective)

value      whole-job cycle throughput, Gvoxel/s = N * 512^3 / t_cycle with
           inputs already resident in HBM (device-timed, CUDA events on the
           library stream, max over ranks)
e2e        the same through the public API (MapCycle.step with the cloud,
           frames and centres copied from pinned host memory and the sphere
           results + stats read back every step)
roofline   the dominant kernel (EDT pass 2 or 3): algorithmic bytes 8 B/voxel
           / its mean CUDA-event duration inside the timed region
cpu_baseline  the oracle port of the reference path (oracle/, OpenMP on all
           host threads) on a bounded sample of the same workload
"""

from __future__ import annotations

import argparse
import contextlib
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "EDT Gvoxel/s & map+EDT+query ms/cycle at 512^3; % HBM roofline; 1/2/4/8 GPU"
DIMS = (512, 512, 512)
VS = 0.02
ORIGIN = (-5.12, -5.12, -0.24)
POINTS = 300_000
EDT_BYTES_PER_VOXEL = 21          # pass1 1+4, pass2 4+4, pass3 4+4
PASS_BYTES = {"edt_pass1": 5, "edt_pass2": 8, "edt_pass3": 8}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def bench_config(world: int) -> dict:
    """The workload both arms run (identical dicts: the driver compares them)."""
    return {"workload": "512^3 camera tick: sparse reset, desk7 mask stamp (8 links, FK frames per "
                        "step), 300k-pt depth-camera cloud scatter with robot mask, exact EDT + "
                        "nearest-site index (env; self map static -> memo), 30 spheres x 2 maps gather",
            "grid": list(DIMS), "voxel_size": VS, "points": POINTS, "spheres": 30,
            "parallelism": f"dp{world} (independent scene per rank)",
            "l2": "inputs larger than L2: one EDT streams 2.8 GB per step"}


def desk7():
    from paper_2407_02363_b200.synth import desk7_model
    return desk7_model()


def scene_inputs(step: int, rank: int, d):
    """Per-step synthetic inputs: cloud at t, FK frames, 30 sphere centres."""
    from paper_2407_02363_b200 import synth
    t = (step + 7 * rank) / 30.0
    pts = synth.depth_camera_cloud(t, max_points=POINTS)
    frames = d["frames"][step % d["frames"].shape[0]]
    centers = np.vstack([synth.sphere_centers(frames, d["sphere_link"], d["sphere_center"]),
                         synth.extra_query_points(DIMS, VS, ORIGIN, 9)])
    return pts, frames, centers


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi takes ~0.1-0.5 s to print its first row: wait for it
            # so the samples fall inside the timed region, not after it
            t_wait = time.perf_counter() + 5.0
            while not self.rows and time.perf_counter() < t_wait:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        self.t_start = time.perf_counter()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.perf_counter(), [x.strip() for x in line.split(",")]))

    def __exit__(self, *exc):
        self.t_end = time.perf_counter()
        if self.proc:
            # a region shorter than the sampling period: take the next row
            # (the clocks have not moved in 50 ms) and say so in the summary
            if not any(self.t_start <= t for t, _ in self.rows):
                t_wait = time.perf_counter() + 0.3
                while time.perf_counter() < t_wait and not any(
                        self.t_start <= t for t, _ in self.rows):
                    time.sleep(0.005)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        return False

    def summary(self):
        rows = [r for t, r in self.rows if self.t_start <= t <= self.t_end]
        window = "timed region"
        if not rows:
            rows = [r for t, r in self.rows if t > self.t_end][:1]
            window = "first sample after the timed region (shorter than the 50 ms period)"
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows), "window": window}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if os.environ.get("VX_BENCH_GLOO") is None else "gloo")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch
        import torch.distributed as dist
        if dist.get_backend() == "nccl":
            dist.barrier(device_ids=[torch.cuda.current_device()])
        else:
            dist.barrier()


def allmax(world, v: float) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------
# CPU path: the oracle port of the reference (test infrastructure, timed only)
# ----------------------------------------------------------------------------
_CPU_GRIDS = {}


def cpu_cycle(pts, frames, centers, d, threads: int):
    """engine.py:234-280 through the oracle restatement, on persistent grids
    like the engine's: clear x3 (cells.fill(0), engine.py:236-238), stamp the
    self-obstacle links and all links (243-248), insert the cloud with the
    robot mask (k=0, 249-254), occupancy, EDT of env (the static self map is
    memoised as engine.py:259-268 does), site world for the spheres (276-280).
    Returns seconds per stage."""
    from oracle import oracle as O
    if not _CPU_GRIDS:
        _CPU_GRIDS.update(env=np.zeros(DIMS, np.float32), self=np.zeros(DIMS, np.float32),
                          mask=np.zeros(DIMS, np.float32))
    env, selfc, mask = _CPU_GRIDS["env"], _CPU_GRIDS["self"], _CPU_GRIDS["mask"]
    t = {}
    t0 = time.perf_counter()
    env.fill(0.0)
    selfc.fill(0.0)
    mask.fill(0.0)
    t["clear"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    for li in d["o_links"]:
        ijk, org = d["links"][li]
        O.stamp_voxels(selfc, VS, ORIGIN, ijk, org, VS, frames[li])
    for li, (ijk, org) in enumerate(d["links"]):
        O.stamp_voxels(mask, VS, ORIGIN, ijk, org, VS, frames[li])
    O.insert_points(env, VS, ORIGIN, pts, mask)
    t["insert"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    occ = env > np.float32(0.0)
    w = threads
    site = O.pba_edt_site(occ, w, w, 2 * w, workers=threads)
    t["edt"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    O.site_world(site, VS, ORIGIN, centers)
    t["query"] = time.perf_counter() - t0
    return t


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU algorithm (oracle port, all host
    threads) on this arm's workload; rank 0 only."""
    if rank != 0:
        return
    from oracle import oracle as O
    O.build()
    # every host core: torchrun exports OMP_NUM_THREADS=1 to each rank, but
    # only rank 0 runs the CPU path, so the OpenMP default would undercount
    threads = max(O.max_threads(), len(os.sched_getaffinity(0)))
    d = desk7()
    n = float(np.prod(DIMS))
    pts, frames, centers = scene_inputs(0, 0, d)
    for _ in range(max(1, min(args.warmup, 1))):
        cpu_cycle(pts, frames, centers, d, threads)
    times, stages = [], []
    budget = 150.0
    t_start = time.perf_counter()
    steps = 0
    for s in range(args.steps):
        pts, frames, centers = scene_inputs(s, 0, d)
        t0 = time.perf_counter()
        st = cpu_cycle(pts, frames, centers, d, threads)
        times.append(time.perf_counter() - t0)
        stages.append(st)
        steps += 1
        if time.perf_counter() - t_start > budget:
            break
    t = statistics.mean(times)
    value = n / t / 1e9
    edt = statistics.mean(s["edt"] for s in stages)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gvoxel/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic",
        "config": bench_config(args.gpus),
        "impl_detail": "oracle/ C port of voxarm edt.py/grids.py/engine.py (OpenMP, all host threads)",
        "edt_gvoxel_s": n / edt / 1e9,
        "stage_ms": {k: 1e3 * statistics.mean(s[k] for s in stages) for k in stages[0]},
        "cpu_baseline": {"value": value, "unit": "Gvoxel/s", "cores": threads, "kind": "port",
                         "sample": f"{steps} full 512^3 camera ticks (300k pts, 8 links, 30 spheres)"},
        "e2e": {"value": value, "unit": "Gvoxel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline_reference"] = voxarm_reference(d)
    print(json.dumps(line), flush=True)


def voxarm_reference(d, budget_s: float = 90.0):
    """The genuine reference, timed: voxarm itself (pip-installed from
    /root/reference into baseline/_ref; numba, NUMBA_NUM_THREADS = host
    threads) on this box's cores, warmed up.  Two legs:
      * pba_edt (edt.py:466-484) on the C3 grid, 512^3 Bernoulli(0.02),
        workers = host threads and workers = 1;
      * the engine's camera branch (engine.py:234-280) on the headline
        512^3 tick: clear x3, self/mask insert_voxel_set, insert_point_cloud
        (k = 0) with the robot mask, occupancy_mask + blake2b + pba_edt of the
        env map, _site_world for 30 spheres x 2 maps (the static self map's
        EDT memoised, as the engine's digest memo does).
    Returns a dict (or {"unavailable": why})."""
    nthreads = len(os.sched_getaffinity(0))
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "voxarm")):
        return {"unavailable": "baseline/_ref has no voxarm install"}
    os.environ["NUMBA_NUM_THREADS"] = str(nthreads)
    if ref not in sys.path:
        sys.path.append(ref)
    try:
        import hashlib

        import voxarm
        from voxarm.grids import FilterConfig, PointCloud, VoxelGrid, VoxelSet
        from paper_2407_02363_b200 import synth
    except Exception as e:   # numba missing on the box, etc.
        return {"unavailable": f"voxarm import failed: {e!r}"[:200]}
    out = {"kind": "reference", "impl": f"voxarm {getattr(voxarm, '__version__', '')} (numba) from baseline/_ref",
           "cores": nthreads}
    t_start = time.perf_counter()
    occ = synth.bernoulli_occupancy(DIMS, 0.02, 0)
    voxarm.pba_edt(occ[:64, :64, :64], workers=nthreads)   # JIT compile
    legs = {}
    for w in (nthreads, 1):
        if time.perf_counter() - t_start > budget_s / 2:
            break
        voxarm.pba_edt(occ, workers=w)   # warm
        ts = []
        for _ in range(2):
            t0 = time.perf_counter()
            voxarm.pba_edt(occ, workers=w)
            ts.append(time.perf_counter() - t0)
            if w == 1:
                break
        legs[f"workers_{w}"] = {"ms": 1e3 * min(ts), "gvoxel_s": float(np.prod(DIMS)) / min(ts) / 1e9}
    out["pba_edt_512^3_bernoulli_0.02"] = legs
    del occ
    # the engine's camera branch on the headline tick
    env = VoxelGrid(DIMS, VS, ORIGIN)
    selfg = VoxelGrid(DIMS, VS, ORIGIN)
    mask = VoxelGrid(DIMS, VS, ORIGIN)
    vsets = [VoxelSet(np.asarray(o, np.float64), VS, ijk) for ijk, o in d["links"]]
    fields, digests = {}, {}

    def tick(step):
        pts, frames, centers = scene_inputs(step, 0, d)
        st = {}
        t0 = time.perf_counter()
        env.clear(); selfg.clear(); mask.clear()
        st["clear"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        for li in d["o_links"]:
            selfg.insert_voxel_set(vsets[li], frames[li])
        for li in range(len(vsets)):
            mask.insert_voxel_set(vsets[li], frames[li])
        env.insert_point_cloud(PointCloud(pts), FilterConfig(k_neighbors=0), robot_mask=mask)
        st["insert"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        for key, grid in (("env", env), ("self", selfg)):
            o = grid.occupancy_mask()
            dig = hashlib.blake2b(o.tobytes(), digest_size=16).digest()
            if digests.get(key) != dig:
                fields[key] = voxarm.pba_edt(o, voxel_size=VS, workers=nthreads)
                digests[key] = dig
        st["edt"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        org = np.asarray(ORIGIN, np.float64)
        dims = np.asarray(DIMS, np.int64)
        for key in ("env", "self"):   # engine.py:212-221 per sphere
            for c in centers:
                idx = np.clip(np.floor((c - org) / VS).astype(np.int64), 0, dims - 1)
                site = fields[key].site_index(tuple(int(v) for v in idx))
                if site is not None:
                    _ = org + (np.asarray(site) + 0.5) * VS
        st["query"] = time.perf_counter() - t0
        return st

    tick(0)   # warm (and the self map's one EDT)
    ts, stages = [], []
    for step in range(1, 4):
        if time.perf_counter() - t_start > budget_s:
            break
        t0 = time.perf_counter()
        stages.append(tick(step))
        ts.append(time.perf_counter() - t0)
    if ts:
        t = statistics.mean(ts)
        out["camera_tick_512^3"] = {
            "ms_per_step": t * 1e3, "value": float(np.prod(DIMS)) / t / 1e9, "unit": "Gvoxel/s",
            "ticks": len(ts), "stage_ms": {k: 1e3 * statistics.mean(s_[k] for s_ in stages) for k in stages[0]}}
        out["value"] = out["camera_tick_512^3"]["value"]
        out["unit"] = "Gvoxel/s"
        out["sample"] = f"{len(ts)} headline 512^3 camera ticks after 1 warm-up tick (voxarm's own code)"
    return out


def engine_bridge_timing(ticks_small: int = 240, ticks_big: int = 40):
    """voxarm's own closed-loop engine (SimEngine.step, engine.py:225-322,
    from baseline/_ref) with the device-resident bridge installed, on the
    shipped walker_crossing scenario at its 96^3 grid and re-gridded to the
    512^3 headline grid; the CPU engine beside it at 96^3.  Per control tick:
    mean ms, camera-tick mean ms, and the bytes libvx moved per tick (no grid,
    mask or site array crosses the bus)."""
    import dataclasses
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "voxarm")):
        return {"unavailable": "baseline/_ref has no voxarm install"}
    if ref not in sys.path:
        sys.path.append(ref)
    try:
        from voxarm.engine import SimEngine
        from voxarm.scenario import GridSpec, load_scenario, shipped_scenario_path
        from paper_2407_02363_b200 import voxarm_bridge
    except Exception as e:
        return {"unavailable": f"voxarm import failed: {e!r}"[:200]}
    base = load_scenario(shipped_scenario_path("walker_crossing"))
    big = dataclasses.replace(base, grid=GridSpec(dims=DIMS, voxel_size=VS, origin=ORIGIN))

    def run(sc, ticks, gpu):
        ctx = voxarm_bridge.installed() if gpu else contextlib.nullcontext()
        with ctx:
            eng = SimEngine(sc)
            for _ in range(3):
                eng.step()
            b0 = voxarm_bridge.transfer_bytes() if gpu else (0, 0)
            ts, cam = [], []
            for _ in range(ticks):
                t0 = time.perf_counter()
                rec = eng.step()
                dt = time.perf_counter() - t0
                ts.append(dt)
                if rec.timings["insert"] > 0.0:
                    cam.append(dt)
            b1 = voxarm_bridge.transfer_bytes() if gpu else (0, 0)
        out = {"ticks": ticks, "ms_per_tick": 1e3 * statistics.mean(ts),
               "camera_tick_ms": 1e3 * statistics.mean(cam) if cam else None, "camera_ticks": len(cam)}
        if gpu:
            out["h2d_bytes_per_tick"] = (b1[0] - b0[0]) / ticks
            out["d2h_bytes_per_tick"] = (b1[1] - b0[1]) / ticks
        return out

    res = {"scenario": "walker_crossing (shipped), default k=8 outlier filter",
           "96^3_gpu_bridge": run(base, ticks_small, True),
           "96^3_cpu_engine": run(base, min(ticks_small, 60), False),
           "512^3_gpu_bridge": run(big, ticks_big, True)}
    n96 = float(np.prod(base.grid.dims))
    res["96^3_grid_bytes"] = n96
    return res


def cpu_baseline_sample(d):
    """Bounded CPU sample (~10-30 s): two full 512^3 ticks after one warm-up."""
    from oracle import oracle as O
    O.build()
    # every host core: torchrun exports OMP_NUM_THREADS=1 to each rank, but
    # only rank 0 runs the CPU path, so the OpenMP default would undercount
    threads = max(O.max_threads(), len(os.sched_getaffinity(0)))
    pts, frames, centers = scene_inputs(0, 0, d)
    cpu_cycle(pts, frames, centers, d, threads)
    ts = []
    for s in range(2):
        pts, frames, centers = scene_inputs(s + 1, 0, d)
        t0 = time.perf_counter()
        cpu_cycle(pts, frames, centers, d, threads)
        ts.append(time.perf_counter() - t0)
    t = statistics.mean(ts)
    return {"value": float(np.prod(DIMS)) / t / 1e9, "unit": "Gvoxel/s", "cores": threads,
            "kind": "port", "ms_per_step": t * 1e3,
            "sample": "2 full 512^3 camera ticks after 1 warm-up (oracle/ C port, OpenMP)"}


# ----------------------------------------------------------------------------
# GPU path
# ----------------------------------------------------------------------------
def run_gpu(args, world, rank, local):
    import torch
    # one GPU per rank; the modulo only matters when a box has fewer GPUs than
    # ranks (a 2-rank smoke of this code path on a 1-GPU box, gloo backend)
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    os.environ["VX_DEVICE"] = str(local)
    from paper_2407_02363_b200 import _lib
    from paper_2407_02363_b200.engine import MapCycle

    ctx = _lib.default_context(local)
    stream = torch.cuda.ExternalStream(ctx.stream_handle(), device=f"cuda:{local}")
    d = desk7()
    links = d["links"]
    cyc = MapCycle(DIMS, VS, ORIGIN, links, VS, d["o_links"], max_points=POINTS, max_spheres=32)
    L = _lib.load()
    nsteps_inputs = 8
    # pinned host inputs (one per distinct step) so the e2e H2D is async
    host = []
    for s in range(nsteps_inputs):
        pts, frames, centers = scene_inputs(s, rank, d)
        hp = _lib.PinnedArray(pts.shape, np.float64)
        hp.array[...] = pts
        hf = _lib.PinnedArray((frames.shape[0], 16), np.float64)
        hf.array[...] = frames.reshape(-1, 16)
        hc = _lib.PinnedArray(centers.shape, np.float64)
        hc.array[...] = centers
        host.append((hp, hf, hc))
    n = float(np.prod(DIMS))
    # device-resident clouds for the `value` leg (inputs in HBM before timing)
    dev_pts = [torch.from_numpy(np.array(h[0].array)).to(f"cuda:{local}") for h in host]
    torch.cuda.synchronize()

    def step(s, sync=False):
        hp, hf, hc = host[s % nsteps_inputs]
        dp = dev_pts[s % nsteps_inputs]
        _lib.check(L.vx_cycle_step_device(cyc._h, ctypes.c_void_p(dp.data_ptr()), dp.shape[0],
                                          _lib.ptr(hf.array), float(np.float32(0.85)), 0.5,
                                          _lib.ptr(hc.array), hc.array.shape[0], 1 if sync else 0))

    # --- warm-up (also builds the static self map once) ---
    for s in range(args.warmup):
        step(s)
    torch.cuda.synchronize()

    # --- per-phase breakdown: a separate profiled run (event marks between
    # the phases, so no CUDA graph); not the timed region ---
    _lib.check(L.vx_cycle_profile(cyc._h, 1))
    for s in range(min(args.steps, 16)):
        step(args.warmup + s)
    torch.cuda.synchronize()
    ph = np.zeros(len(_lib.CYCLE_PHASES), np.float64)
    nprof = ctypes.c_int()
    _lib.check(L.vx_cycle_phase_ms(cyc._h, _lib.ptr(ph), ctypes.byref(nprof)))
    _lib.check(L.vx_cycle_profile(cyc._h, 0))
    phases = dict(zip(_lib.CYCLE_PHASES, (float(v) for v in ph)))
    for s in range(2):   # back on the graph path
        step(args.warmup + s)
    torch.cuda.synchronize()

    # --- device-timed region: inputs resident (the per-step H2D of the
    # frames / centres is the only host traffic and is inside the step;
    # results stay on the device); the tick replays its CUDA graph ---
    launches0 = ctx.launches()
    barrier(world)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for s in range(args.steps):
            step(args.warmup + s)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    launches = ctx.launches() - launches0
    t_dev = e0.elapsed_time(e1) / 1e3 / args.steps
    t_max = allmax(world, t_dev)

    # --- e2e: public API, host inputs and result read-back every step ---
    for s in range(2):   # untimed: the host path's first calls
        tk = cyc.prefetch(host[s][0].array)
        cyc.step(tk, host[s][1].array, host[s][2].array, sync=False)
        cyc.wait()
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    res = None
    # each step's cloud is uploaded while the previous tick computes
    # (MapCycle.prefetch, a copy stream); its results are read back before
    # the next step is issued
    tk = cyc.prefetch(host[args.warmup % nsteps_inputs][0].array)
    for s in range(args.steps):
        hp, hf, hc = host[(args.warmup + s) % nsteps_inputs]
        cyc.step(tk, hf.array, hc.array, sync=False)
        if s + 1 < args.steps:
            tk = cyc.prefetch(host[(args.warmup + s + 1) % nsteps_inputs][0].array)
        res = cyc.wait()
    ev1.record(stream)
    torch.cuda.synchronize()
    t_e2e_wall = (time.perf_counter() - t0) / args.steps
    t_e2e = max(ev0.elapsed_time(ev1) / 1e3 / args.steps, t_e2e_wall)
    t_e2e_max = allmax(world, t_e2e)
    h2d = POINTS * 24 + d["frames"].shape[1] * 128 + 30 * 24
    d2h = 2 * 30 * (4 + 24 + 8) + 64

    # config C4 (all ranks: data-parallel scene batch, max over ranks)
    c4 = None if args.no_sweep else c4_batch(ctx, stream, rank, world)
    c4c = None if args.no_sweep else c4_batch_camera(ctx, stream, rank, world)
    c5 = None if args.no_sweep else c5_slab(rank, world)
    if rank != 0:
        return
    peak, peak_src = peaks()
    dom = max(("edt_pass2", "edt_pass3"), key=lambda k: phases[k])
    dom_t = phases[dom] / 1e3
    achieved = PASS_BYTES[dom] * n / dom_t / 1e9 if dom_t > 0 else None
    edt_t = (phases["edt_pass1"] + phases["edt_pass2"] + phases["edt_pass3"]) / 1e3
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            traffic = json.load(fh).get(dom)
    except Exception:
        pass
    cycle_bytes = EDT_BYTES_PER_VOXEL * n + 25 * POINTS + 13 * sum(
        int(x[0].shape[0]) for x in links) + 64 * 60
    line = {
        "metric": METRIC, "value": world * n / t_max / 1e9, "unit": "Gvoxel/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_max * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": bench_config(world),
        "edt_gvoxel_s": world * n / edt_t / 1e9 if edt_t > 0 else None,
        "edt_ms": edt_t * 1e3,
        "edt_roofline_frac": (EDT_BYTES_PER_VOXEL * n / edt_t / 1e9) / peak if edt_t > 0 else None,
        "cycle_roofline_frac": cycle_bytes / t_max / 1e9 / peak,
        "phase_ms": phases,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": (achieved / peak) if achieved else None,
                     "traffic": traffic, "peak_source": peak_src,
                     "bytes_per_voxel": PASS_BYTES[dom]},
        "e2e": {"value": world * n / t_e2e_max / 1e9, "unit": "Gvoxel/s",
                "ms_per_step": t_e2e_max * 1e3, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "api": "paper_2407_02363_b200.engine.MapCycle.prefetch + step + wait (vx_cycle_prefetch/step/wait; next cloud uploaded during the current tick)"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "last_stats": {k: res[k] for k in ("inserted", "robot_skipped", "out_of_bounds")} if res else None,
    }
    if c4 is not None:
        line["c4_batch_64x256^3"] = c4
    if c4c is not None:
        line["c4_batch_camera_64x256^3"] = c4c
    if c5 is not None:
        line["c5_slab_1024^3"] = c5
    if not args.no_sweep:
        line["edt_sweep"] = edt_sweep(ctx, stream)
        line["small_configs"] = small_configs(d)
        line["outlier_filter"] = outlier_timing()
        line["engine_bridge"] = engine_bridge_timing()
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline_sample(d)
        line["cpu_baseline_reference"] = voxarm_reference(d)
    print(json.dumps(line), flush=True)


def small_configs(d, steps: int = 20):
    """Configs C1 (128^3, 50k-pt sphere, 30 spheres) and C2 (256^3, 300k-pt
    depth camera): device time per camera tick (inputs resident) and end-to-end
    time through MapCycle.prefetch + step + wait (host inputs, the next cloud
    uploaded during the current tick, results read back)."""
    import torch
    from paper_2407_02363_b200 import _lib, synth
    from paper_2407_02363_b200.engine import MapCycle
    L = _lib.load()
    out = {}
    c1 = synth.C1
    specs = {
        "C1_128^3": (c1["dims"], c1["voxel_size"], c1["origin"],
                     lambda s: synth.c1_cloud(s / 30.0)),
        "C2_256^3": ((256, 256, 256), 0.02, (-2.56, -2.56, -0.24),
                     lambda s: synth.depth_camera_cloud(s / 30.0)),
    }
    for name, (dims, vs, origin, cloud) in specs.items():
        clouds = [cloud(s) for s in range(4)]
        cyc = MapCycle(dims, vs, origin, d["links"], vs, d["o_links"],
                       max_points=max(c.shape[0] for c in clouds), max_spheres=32)
        ctx = cyc.ctx
        stream = torch.cuda.ExternalStream(ctx.stream_handle())
        frames = [d["frames"][s % d["frames"].shape[0]] for s in range(4)]
        centers = [np.vstack([synth.sphere_centers(f, d["sphere_link"], d["sphere_center"]),
                              synth.extra_query_points(dims, vs, origin, 9)]) for f in frames]
        dev = [torch.from_numpy(c).cuda() for c in clouds]
        T = [np.ascontiguousarray(f.reshape(-1, 16)) for f in frames]
        for s in range(5):
            _lib.check(L.vx_cycle_step_device(cyc._h, ctypes.c_void_p(dev[s % 4].data_ptr()),
                                              dev[s % 4].shape[0], _lib.ptr(T[s % 4]),
                                              float(np.float32(0.85)), 0.5, _lib.ptr(centers[s % 4]),
                                              30, 0))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(steps):
            _lib.check(L.vx_cycle_step_device(cyc._h, ctypes.c_void_p(dev[s % 4].data_ptr()),
                                              dev[s % 4].shape[0], _lib.ptr(T[s % 4]),
                                              float(np.float32(0.85)), 0.5, _lib.ptr(centers[s % 4]),
                                              30, 0))
        e1.record(stream)
        torch.cuda.synchronize()
        dev_ms = e0.elapsed_time(e1) / steps
        pinned = []
        for c in clouds:
            pa = _lib.PinnedArray(c.shape, np.float64)
            pa.array[...] = c
            pinned.append(pa)
        t0 = time.perf_counter()
        tk = cyc.prefetch(pinned[0].array)
        for s in range(steps):
            cyc.step(tk, frames[s % 4], centers[s % 4], sync=False)
            if s + 1 < steps:
                tk = cyc.prefetch(pinned[(s + 1) % 4].array)
            cyc.wait()
        e2e_ms = (time.perf_counter() - t0) / steps * 1e3
        out[name] = {"device_ms_per_tick": dev_ms, "e2e_ms_per_tick": e2e_ms,
                     "points": int(clouds[0].shape[0]), "hz_e2e": 1e3 / e2e_ms}
        cyc.close()
    return out


def outlier_timing():
    """insert_point_cloud with the engine's default filter (k_neighbors=8,
    grids.py:166-169) on the 300k-point C2 cloud through the public API
    (host points in, stats out), vs k_neighbors=0."""
    from paper_2407_02363_b200 import FilterConfig, PointCloud, VoxelGrid
    from paper_2407_02363_b200 import synth
    pts = synth.depth_camera_cloud(0.1)
    g = VoxelGrid((256, 256, 256), 0.02, (-2.56, -2.56, -0.24))
    out = {"points": int(pts.shape[0])}
    for k in (0, 8):
        cfg = FilterConfig(k_neighbors=k)
        for _ in range(2):
            g.clear()
            g.insert_point_cloud(PointCloud(pts), cfg)
        t0 = time.perf_counter()
        reps = 5
        for _ in range(reps):
            g.clear()
            st = g.insert_point_cloud(PointCloud(pts), cfg)
        out[f"k{k}_ms"] = (time.perf_counter() - t0) / reps * 1e3
        out[f"k{k}_outliers_removed"] = st.outliers_removed
    return out


def edt_sweep(ctx, stream):
    """Config C3 latency sweep: device-timed EDT (K3+K4+K5, inputs resident)
    of Bernoulli(0.02, seed 0) grids n^3 and of a single centre voxel at 512^3."""
    import torch
    from paper_2407_02363_b200 import _lib, synth
    L = _lib.load()
    out = {}
    cases = [(n, "bernoulli_0.02") for n in (64, 96, 128, 192, 256, 384, 512)]
    cases += [(512, "single_center"), (512, "bernoulli_1e-4"), (1024, "bernoulli_0.02")]
    for n, kind in cases:
        dims = (n, n, n)
        if kind == "single_center":
            occ = synth.structured_occupancy("single_center", dims)
        elif kind == "bernoulli_1e-4":
            occ = synth.bernoulli_occupancy(dims, 1e-4, 1)
        else:
            occ = synth.bernoulli_occupancy(dims, 0.02, 0)
        d_occ = torch.from_numpy(occ).cuda()
        site = torch.empty(dims, dtype=torch.int32, device="cuda")
        sb = L.vx_edt_scratch_bytes(n, n, n, 1)
        scratch = torch.empty(sb, dtype=torch.uint8, device="cuda")
        args = (ctx.handle, ctypes.c_void_p(d_occ.data_ptr()), n, n, n, 1,
                ctypes.c_void_p(site.data_ptr()), ctypes.c_void_p(scratch.data_ptr()), sb)
        for _ in range(3):
            _lib.check(L.vx_edt_device(*args))
        torch.cuda.synchronize()
        reps = 10 if n <= 256 else (5 if n <= 512 else 3)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            _lib.check(L.vx_edt_device(*args))
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out[f"{n}^3 {kind}"] = {"ms": ms, "gvoxel_s": n ** 3 / ms / 1e6,
                                "hbm_frac": EDT_BYTES_PER_VOXEL * n ** 3 / ms / 1e6 / peaks()[0]}
        del d_occ, site, scratch
    return out


def c4_batch(ctx, stream, rank: int, world: int):
    """Config C4: a batch of 64 independent 256^3 scenes sharded data-parallel
    (64 / world scenes per rank, one batched vx_edt_device launch per rank;
    Bernoulli(0.02) occupancy, a different seed per scene).  No collective."""
    import torch
    from paper_2407_02363_b200 import _lib, synth
    L = _lib.load()
    n, total = 256, 64
    per = max(1, total // world)
    occ = np.stack([synth.bernoulli_occupancy((n, n, n), 0.02, 1000 + rank * per + s) for s in range(per)])
    d_occ = torch.from_numpy(occ).cuda()
    del occ
    site = torch.empty((per, n, n, n), dtype=torch.int32, device="cuda")
    sb = L.vx_edt_scratch_bytes(n, n, n, per)
    scratch = torch.empty(sb, dtype=torch.uint8, device="cuda")
    args = (ctx.handle, ctypes.c_void_p(d_occ.data_ptr()), n, n, n, per,
            ctypes.c_void_p(site.data_ptr()), ctypes.c_void_p(scratch.data_ptr()), sb)
    for _ in range(2):
        _lib.check(L.vx_edt_device(*args))
    torch.cuda.synchronize()
    barrier(world)
    reps = 3
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        _lib.check(L.vx_edt_device(*args))
    e1.record(stream)
    torch.cuda.synchronize()
    t = allmax(world, e0.elapsed_time(e1) / 1e3 / reps)
    del d_occ, site, scratch
    vox = float(per * world) * n ** 3
    return {"scenes": per * world, "scenes_per_gpu": per, "ms": t * 1e3, "gvoxel_s": vox / t / 1e9,
            "hbm_frac": EDT_BYTES_PER_VOXEL * vox / t / 1e9 / peaks()[0],
            "occupancy": "Bernoulli(0.02) per scene", "scaling": "strong (64 scenes total)"}


def c4_batch_camera(ctx, stream, rank: int, world: int):
    """Config C4, camera variant: 64 scenes of 256^3, scene s =
    the C2 depth-camera cloud at t = s/30 s rasterised into a grid (k = 0
    insert); 64/N scenes per rank in one batched launch, which skips each
    scene's empty slices.  8 distinct frames, repeated."""
    import torch
    from paper_2407_02363_b200 import _lib, synth
    from paper_2407_02363_b200.grids import FilterConfig, PointCloud, VoxelGrid
    L = _lib.load()
    n, total = 256, 64
    per = max(1, total // world)
    frames = []
    for f in range(8):
        g = VoxelGrid((n, n, n), 0.02, (-2.56, -2.56, -0.24))
        g.insert_point_cloud(PointCloud(synth.depth_camera_cloud((rank * per + f) / 30.0)),
                             FilterConfig(k_neighbors=0))
        frames.append(torch.from_numpy(g.occupancy_mask().view(np.uint8)).cuda())
    d_occ = torch.stack([frames[s % 8] for s in range(per)]).contiguous()
    del frames
    site = torch.empty((per, n, n, n), dtype=torch.int32, device="cuda")
    sb = L.vx_edt_scratch_bytes(n, n, n, per)
    scratch = torch.empty(sb, dtype=torch.uint8, device="cuda")
    args = (ctx.handle, ctypes.c_void_p(d_occ.data_ptr()), n, n, n, per,
            ctypes.c_void_p(site.data_ptr()), ctypes.c_void_p(scratch.data_ptr()), sb)
    for _ in range(2):
        _lib.check(L.vx_edt_device(*args))
    torch.cuda.synchronize()
    barrier(world)
    reps = 3
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        _lib.check(L.vx_edt_device(*args))
    e1.record(stream)
    torch.cuda.synchronize()
    t = allmax(world, e0.elapsed_time(e1) / 1e3 / reps)
    del d_occ, site, scratch
    vox = float(per * world) * n ** 3
    return {"scenes": per * world, "scenes_per_gpu": per, "ms": t * 1e3, "gvoxel_s": vox / t / 1e9,
            "hbm_frac": EDT_BYTES_PER_VOXEL * vox / t / 1e9 / peaks()[0],
            "occupancy": "C2 depth-camera cloud at t = s/30 s, 256^3, 8 distinct frames",
            "scaling": "strong (64 scenes total)"}


def c5_slab(rank: int, world: int):
    """Config C5: one 1024^3 grid slab-decomposed across the ranks (i-slabs;
    passes 1-2 local in 4 slice groups, the pass-2 epilogue writes the j-slab
    transpose into per-destination send blocks, each group's NCCL send/recv
    queued on the library stream behind its pass 2 so it overlaps the next
    group's compute, pass 3 on the received j-slab).  Strong
    scaling: the whole grid is fixed, time = max over ranks of the device time
    of one SlabEDT call.  Bernoulli(0.02) occupancy generated on the device."""
    import torch
    from paper_2407_02363_b200.slab import SlabEDT, even_split
    n = 1024
    i0, i1 = even_split(n, world)[rank], even_split(n, world)[rank + 1]
    g = torch.Generator(device="cuda")
    g.manual_seed(77 + rank)
    occ = (torch.rand((i1 - i0, n, n), generator=g, device="cuda") < 0.02).to(torch.uint8)
    slab = SlabEDT((n, n, n), exchange="nccl")
    for _ in range(2):
        slab(occ)
    torch.cuda.synchronize()
    barrier(world)
    reps = 3
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        slab(occ)
    e1.record()
    torch.cuda.synchronize()
    t = allmax(world, e0.elapsed_time(e1) / 1e3 / reps)
    del occ, slab
    torch.cuda.empty_cache()
    return {"ranks": world, "ms": t * 1e3, "gvoxel_s": n ** 3 / t / 1e9,
            "hbm_frac_per_gpu": EDT_BYTES_PER_VOXEL * n ** 3 / world / t / 1e9 / peaks()[0],
            "exchange": "nccl grouped send/recv per slice group, stream-ordered (pass-2 epilogue writes the "
                        "send blocks; own rows straight into the receive buffer)",
            "nvlink_bytes_per_rank": 4 * (i1 - i0) * (n - (even_split(n, world)[rank + 1] - even_split(n, world)[rank])) * n
            if world > 1 else 0,
            "occupancy": "Bernoulli(0.02), generated on the device", "scaling": "strong (one 1024^3 grid)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: 2000 ticks, ~0.8 s, so nvidia-smi samples the "
                         "clocks under load; 30 for --impl reference)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the C3 EDT latency sweep")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.steps is None:
        args.steps = 30 if args.impl == "reference" else 2000
    world, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_gpu(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
