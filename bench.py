#!/usr/bin/env python
"""Benchmark: wavelet analysis+synthesis round trips/s (BASELINE.json metric).

Default workload (N=1): BASELINE config C4 -- L=2048 MW sampling, one complex
map with f_lm ~ Gaussian, C_l = (l+1)^-2, lambda=3, J0=2, multiresolution.
One step = one wavelet analysis + synthesis round trip of the map.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

N > 1 runs under torchrun and, by default, partitions the ONE map of the
config over the ranks as BASELINE C4/C5 name it (--mode shard: orders m for
the Legendre/theta stages, theta rings for the phi stages, NCCL all-to-all
between them; small scale bands placed whole on one rank; "scaling":
"strong").  --mode replica runs one independent map per rank ("weak").
Timing is the max over ranks of CUDA-event time.
--impl reference times the CPU oracle port of the same path (oracle/, C with
OpenMP, the reference itself being pure Python that cannot leave this repo's
build container) on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "wavelet analysis+synthesis round-trips/s at L=2048; FP64 peak and HBM fraction"

# BASELINE.json configs (SURVEY 8(d) spectra)
CONFIGS = {
    "C1": dict(L=64, batch=1, real=False, lam=2.0, j0=0, multires=False, spec="flat"),
    "C2": dict(L=256, batch=16, real=True, lam=2.0, j0=2, multires=True, spec="cl"),
    "C3": dict(L=1024, batch=8, real=False, lam=2.0, j0=3, multires=True, spec="flat"),
    "C4": dict(L=2048, batch=1, real=False, lam=3.0, j0=2, multires=True, spec="l1"),
    "C5": dict(L=4096, batch=1, real=True, lam=2.0, j0=0, multires=True, spec="beam"),
}


def _executed(cfgname, kernel, mode):
    """Executed FP64 (+ DMMA) pipe utilisation of the roofline stage from the
    committed ncu capture (profiles/roofline_traffic.json), or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                        "roofline_traffic.json")
    if mode == "shard" or not os.path.exists(path):
        return None, None
    try:
        with open(path) as fh:
            rec = json.load(fh).get(cfgname, {}).get(kernel)
        return (float(rec["executed_pipe_frac"]), rec.get("executed_note")) if rec else (None, None)
    except (OSError, ValueError, KeyError):
        return None, None


def _traffic(cfgname, kernel, mode):
    """DRAM bytes per launch of the roofline kernel from the committed ncu capture
    (profiles/roofline_traffic.json), or None when none matches this workload."""
    import json

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                        "roofline_traffic.json")
    if mode == "shard" or not os.path.exists(path):
        return None
    try:
        with open(path) as fh:
            rec = json.load(fh).get(cfgname, {}).get(kernel)
        return int(rec["dram_bytes_per_launch"]) if rec else None
    except (OSError, ValueError, KeyError):
        return None


def spectrum(name, L):
    ell = np.arange(L, dtype=np.float64)
    if name == "flat":
        return np.ones(L)
    if name == "l1":
        return (ell + 1.0) ** -2
    base = np.where(ell >= 2, 1.0 / np.maximum(ell * (ell + 1.0), 1.0), 0.0)
    if name == "cl":
        return base
    sigma = 5.0 / 60.0 * np.pi / 180.0
    return base * np.exp(-ell * (ell + 1.0) * sigma**2 / 2.0)


def seeded_coeffs(L, real, spec, seed):
    from paper_1211_1680_b200 import gaussian_coeffs

    f = gaussian_coeffs(L, np.random.default_rng(seed), real_signal=real)
    ell = np.repeat(np.arange(L), 2 * np.arange(L) + 1)
    return f.coeffs * np.sqrt(spectrum(spec, L))[ell]


def legendre_flops(k, nsets, real):
    """Canonical FLOPs of one Legendre stage: 4 B k S + 4 k k(k+1)/2."""
    S = k * (k + 1) / 2 if real else k * k
    return 4.0 * nsets * k * S + 4.0 * k * k * (k + 1) / 2


def hbm_peak_gbs():
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json, driver-written), else the
    B200_PROFILING.md fallback."""
    try:
        with open(ROOT / "MEASURED_PEAKS.json") as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, burst)"
    except (OSError, ValueError, KeyError):
        return 7700.0, "fallback 7.7 TB/s (B200_PROFILING.md)"


def stage_bytes(cfg, bands):
    """Algorithmic HBM bytes per round trip of the ring-FFT and theta stages
    (SURVEY 8(d)): one read of the input and one write of the output per SHT.
    phi: k(2k-1) e + k n_m 16 (e = 8 real / 16 complex map samples; n_m = k
    real / 2k-1 complex Fourier columns); theta (MW forward) and the MW
    synthesis resampling (k >= 1024): 2 k n_m 16.  The SHTs of a round trip run
    at L and at every scale band, once per direction."""
    B, real = cfg["batch"], cfg["real"]
    ks = [cfg["L"]] + list(bands)
    e = 8 if real else 16

    def nm(k):
        return k if real else 2 * k - 1

    phi = sum(B * (k * (2 * k - 1) * e + k * nm(k) * 16) for k in ks)
    theta = sum(B * 2 * k * nm(k) * 16 for k in ks)
    theta += sum(B * 2 * k * nm(k) * 16 for k in ks if k >= 1024)
    return {"phi_fwd": phi, "phi_inv": phi, "theta": theta}


def stage_flops(cfg, bands):
    """Canonical FLOPs per round trip of each Legendre stage.  Analysis
    direction: leg_ana at L, leg_synth over the scale grids; synthesis: the
    mirror.  Divided by the stage's measured time per round trip (not per
    launch: the launch count depends on the path -- grouped, per scale when
    sharded, plus the Reinsch launch of the low orders)."""
    L, B, real = cfg["L"], cfg["batch"], cfg["real"]
    groups = {}
    for k in bands:
        groups[k] = groups.get(k, 0) + B
    grouped = sum(legendre_flops(k, n, real) for k, n in groups.items())
    top = legendre_flops(L, B, real)
    return {"leg_ana": top + grouped, "leg_synth": top + grouped, "per_rt": 2.0 * (top + grouped)}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu, self.rows, self._stop = gpu_index, [], threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=6)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for n, v in zip(names, r[4:8]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_ours(args, cfgname):
    import torch
    import torch.distributed as dist

    import paper_1211_1680_b200 as sw
    from paper_1211_1680_b200 import _native
    from paper_1211_1680_b200 import distributed as D
    from paper_1211_1680_b200.device import SphericalHarmonicTransform, WaveletTransform

    ws, rank, local = dist_env()
    # NCCL's banner / warnings go to stderr: stdout carries the one JSON line
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    torch.cuda.set_device(local)
    mode = args.mode or ("shard" if ws > 1 else "single")
    if ws > 1 or mode == "shard":
        for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29533"), ("RANK", "0"),
                     ("WORLD_SIZE", "1")):
            os.environ.setdefault(k, v)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    cfg = CONFIGS[cfgname]
    L, B, real = cfg["L"], cfg["batch"], cfg["real"]
    scheme = sw.SamplingScheme.MW
    tcfg = sw.TransformConfig(L, cfg["lam"], cfg["j0"], scheme=scheme, multires=cfg["multires"])

    # seeded input (untimed setup): f_lm -> MW map through our own synthesis.
    # single / replica: every rank transforms its own map(s); shard: the ranks
    # share ONE batch of maps, each holding its ring block.
    seed0 = 1000 + (97 * rank if mode == "replica" else 0)
    flm = np.stack([seeded_coeffs(L, real, cfg["spec"], seed0 + b) for b in range(B)])
    sht = SphericalHarmonicTransform(scheme, L)
    x_full = sht.synthesis(torch.from_numpy(flm).cuda(), real=real)
    x_full0 = x_full[0].cpu().numpy()
    st = torch.cuda.current_stream()

    if mode == "shard":
        ex = D.TorchExchange()
        if args.exchange == "peer":
            # fused exchange over NVLink peer memory (CUDA IPC between the ranks);
            # a rank set that cannot map its peers' buffers keeps the NCCL path
            try:
                ex = D.TorchPeerExchange()
                ex.alloc_shared(("probe",), {q: (1,) for q in range(ws)}, torch.float64)
            except Exception as e:  # pragma: no cover - hardware dependent
                print(f"peer exchange unavailable ({e}); using NCCL P2P", file=sys.stderr)
                ex = D.TorchExchange()
        sh = D.ShardedWaveletTransform(tcfg, ex, batch=B, real=real)
        t0, t1 = sh.ring_block(L, rank)
        x = x_full[:, t0:t1, :].contiguous()
        bands = sh.bands

        def step(inp):
            return sh.round_trip({rank: inp})[rank]

        maps_per_step = B  # the job transforms one batch per step
    else:
        wt = WaveletTransform(tcfg, batch=B, real=real)
        x = x_full
        bands = wt.bands
        scale = wt.alloc_scale_maps()
        out_buf = torch.empty_like(x)

        def step(inp):
            return wt.round_trip(inp, scale, out_buf)

        maps_per_step = ws * B
    del x_full

    def barrier():
        if dist.is_initialized():
            dist.barrier()

    out = None
    for _ in range(args.warmup):
        out = step(x)
    torch.cuda.synchronize()
    err = (out - x).abs().max().item() / max(x.abs().max().item(), 1e-300)
    if ws > 1:
        t = torch.tensor([err], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        err = t.item()

    # --- device-resident timed region.  Each step replays a CUDA graph of the
    # round trip (--graph auto/on; small maps are launch-bound) and the
    # per-stage profile comes from a separate eager pass.
    # (auto: always; at L = 2048 the graph removes the GPU-side gaps between the
    # ~40 dependent launches of a round trip, +0.5%; at L <= 512 it is 2x)
    use_graph = mode != "shard" and args.graph in ("on", "auto")
    if use_graph:
        def timed_step(inp):
            return wt.round_trip_graph(inp, scale, out_buf)

        timed_step(x)
    else:
        timed_step = step
    _native.profile_enable(False)
    l0 = _native.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record(st)
        for _ in range(args.steps):
            out = timed_step(x)
        ev1.record(st)
        torch.cuda.synchronize()
        barrier()
    launches = _native.kernel_launches() - l0
    if use_graph:
        # graph replays are not counted by the library: the replay launches the
        # same kernels as one eager round trip
        l1 = _native.kernel_launches()
        step(x)
        torch.cuda.synchronize()
        launches = (_native.kernel_launches() - l1) * args.steps
    # per-stage breakdown (CUDA events around every launch) from a separate
    # eager pass after the timed region, with the per-scale stages serialised
    # on one stream so that stage times add up
    n_prof = max(1, min(args.steps, 5))
    if mode != "shard":
        wt.set_concurrency(False)
    _native.profile_enable(True)
    _native.profile_read(reset=True)
    for _ in range(n_prof):
        step(x)
    torch.cuda.synchronize()
    prof = _native.profile_read(reset=True)
    _native.profile_enable(False)
    if mode != "shard":
        wt.set_concurrency(True)
    ms = ev0.elapsed_time(ev1)
    if ws > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    value = maps_per_step * args.steps / (ms / 1e3)

    # --- end to end through the public API with pinned host buffers: every
    # step copies its map in (H2D) and its reconstruction out (D2H); the
    # single-GPU/replica path streams them (WaveletTransform.round_trip_stream:
    # the copies of neighbouring steps overlap the transforms)
    x_host = x.cpu().pin_memory()
    out_host = [torch.empty_like(x_host).pin_memory() for _ in range(2)]

    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    xin = [torch.empty_like(x) for _ in range(2)]

    def shard_stream(k):
        """The shard path's copies overlapped like round_trip_stream's: the H2D of
        step i+1 and the D2H of step i-1 run on their own streams under step i."""
        ready = [torch.cuda.Event() for _ in range(2)]
        done = [torch.cuda.Event() for _ in range(2)]
        free = [torch.cuda.Event() for _ in range(2)]
        for e in free:
            e.record(st)
        with torch.cuda.stream(h2d_s):
            xin[0].copy_(x_host, non_blocking=True)
            ready[0].record(h2d_s)
        for i in range(k):
            b = i & 1
            if i + 1 < k:
                with torch.cuda.stream(h2d_s):
                    h2d_s.wait_event(free[b ^ 1])
                    xin[b ^ 1].copy_(x_host, non_blocking=True)
                    ready[b ^ 1].record(h2d_s)
            st.wait_event(ready[b])
            y = step(xin[b])
            free[b].record(st)
            done[b].record(st)
            y.record_stream(d2h_s)  # the allocator must not reuse y before the copy
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(done[b])
                out_host[b].copy_(y, non_blocking=True)
        st.wait_stream(d2h_s)
        d2h_s.synchronize()

    def e2e_steps(k):
        if mode == "shard":
            shard_stream(k)
        else:
            wt.round_trip_stream([x_host] * k, [out_host[i & 1] for i in range(k)])

    e2e_steps(max(1, args.warmup // 2))
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    e2e_steps(args.steps)
    e1.record(st)
    torch.cuda.synchronize()
    err_e2e = (out_host[(args.steps - 1) & 1].cuda() - x).abs().max().item() / max(
        x.abs().max().item(), 1e-300)
    if err_e2e > 10 * max(err, 1e-14):
        raise RuntimeError(f"streamed round trip differs from the device round trip ({err_e2e:.3e})")
    ms_e2e = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([ms_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = t.item()
    e2e = maps_per_step * args.steps / (ms_e2e / 1e3)
    nbytes = x.numel() * x.element_size()

    # --- end to end through the numpy drop-in, as the reference's run_trial
    # times it (bench.py:84-92): host SphereMap(s) -> wav_analysis_pixel ->
    # host WaveletDecomposition(s) -> wav_synthesis_pixel -> host SphereMap(s);
    # every scale map crosses PCIe in both directions, synchronously
    dropin = None
    if mode != "shard":
        dropin = dropin_e2e(sw, tcfg, flm, real, args, barrier, ws)
    fp64_peak = _native.fp64_peak_tflops(None)
    dmma_peak = _native.dmma_peak_tflops(None)
    if rank != 0:
        if dist.is_initialized():
            dist.destroy_process_group()
        return None
    fl = stage_flops(cfg, bands)
    dom = max(("leg_synth", "leg_ana"), key=lambda s: prof[s][0])
    dms, dn = prof[dom]
    # per GPU: the job's FLOPs of the stage per round trip / P, over this rank's
    # stage time per round trip (the profile pass ran n_prof round trips)
    shard_frac = 1.0 / ws if mode == "shard" else 1.0
    achieved = (fl[dom] * shard_frac / (dms / n_prof * 1e-3) / 1e12) if dms else None
    peak = max(fp64_peak, dmma_peak)
    stages = {k: {"ms_per_step": v[0] / n_prof, "launches_per_step": v[1] / n_prof}
              for k, v in prof.items()}
    rec = {
        "metric": METRIC,
        "value": value,
        "unit": "round-trips/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if mode == "shard" else "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded Gaussian f_lm, BASELINE spectrum; MW map from our synthesis)",
        "config": workload_config(cfgname, bands, mode, ws,
                                  nbytes * (ws if mode == "shard" else 1)),
        "e2e": {"value": e2e, "unit": "round-trips/s", "h2d_bytes_per_step": nbytes,
                "d2h_bytes_per_step": nbytes,
                "api": ("ShardedWaveletTransform.round_trip (H2D/D2H of neighbouring steps overlap "
                        "the transforms; pinned host buffers)" if mode == "shard" else
                        "WaveletTransform.round_trip_stream (H2D/D2H of neighbouring steps overlap "
                        "the transforms; pinned host buffers)")},
        "e2e_dropin": dropin,
        "gpu_launches": int(launches),
        "cuda_graph": use_graph,
        "roofline": {
            "bound": "fp64", "kernel": dom,
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak if achieved else None,
            "traffic": _traffic(cfgname, dom, mode),
            # canonical FLOPs count the unsymmetrised work; the kernels execute about
            # half of it (equator symmetry), so the hardware view is the pipe utilisation
            "executed_frac": _executed(cfgname, dom, mode)[0],
            "executed_note": _executed(cfgname, dom, mode)[1],
            "traffic_unit": "bytes per launch (DRAM read + write, ncu --set full)",
            "flops_per_rt": fl[dom] * shard_frac,
            "stage_ms_per_rt": dms / n_prof,
            "launches_per_rt": dn / n_prof,
            "peak_source": f"measured in this run: DFMA {fp64_peak:.1f}, DMMA {dmma_peak:.1f} "
                           "TFLOP/s (s2w_fp64_peak / s2w_dmma_peak); MEASURED_PEAKS.json has "
                           "no FP64 entry",
        },
        "stages": stages,
        "stages_note": ("per-stage CUDA-event times from a separate eager pass after the timed "
                        "region with the per-scale stages serialised on one stream; the timed "
                        "region runs them concurrently on forked side streams"),
        "hbm_stages": hbm_stages(cfg, bands, stages),
        "canonical_flops_per_rt": fl["per_rt"],
        "fp64_tflops_per_gpu": fl["per_rt"] * value / ws / 1e12 / B,
        "rt_rel_err": err,
        "clocks": clk.summary(),
    }
    rec["cpu_baseline"] = cpu_baseline(cfgname, args) if not args.no_cpu else None
    if not args.no_cpu:
        rec["parity"] = oracle_parity(cfg, flm[0], x_full0, sht)
    if dist.is_initialized():
        dist.destroy_process_group()
    return rec


def dropin_e2e(sw, tcfg, flm, real, args, barrier, ws):
    """Round trips/s of the drop-in's host API (run_trial's timed pair), wall
    clock around K synchronous steps (each call returns host arrays), max
    over ranks; the batch configs go through the *_batch variants.  As in
    run_trial (reference bench.py:80-83) the input maps come from the drop-in's
    own sh_synthesis of the seeded coefficients, untimed."""
    import torch
    import torch.distributed as dist
    from paper_1211_1680_b200.sht import sh_synthesis_stack

    grid = sw.make_grid(tcfg.scheme, tcfg.L)
    maps = sh_synthesis_stack([sw.HarmonicCoeffs(tcfg.L, f, real_signal=real) for f in flm], grid)
    B = len(maps)

    def one():
        dec = sw.wav_analysis_pixel_batch(maps, tcfg)
        return dec, sw.wav_synthesis_pixel_batch(dec)

    dec, rec = one()
    err = max(float(np.abs(r.values - m.values).max()) for r, m in zip(rec, maps))
    # SphereMap values are complex128 on the host for real maps too (reference grid.py:99-123)
    scale_bytes = sum(m.values.nbytes for d in dec[:1] for m in (d.scaling, *d.wavelets)) * B
    map_bytes = B * maps[0].values.nbytes
    k = max(1, min(args.steps, 10))
    del dec, rec  # their page-locked blocks go back to the host pool, as in a user's loop
    barrier()
    t0 = time.perf_counter()
    for _ in range(k):
        one()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if ws > 1:
        t = torch.tensor([dt], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = t.item()
    return {"value": ws * B * k / dt, "unit": "round-trips/s", "steps": k,
            "h2d_bytes_per_step": map_bytes + scale_bytes, "d2h_bytes_per_step": scale_bytes + map_bytes,
            "max_abs_err": err,
            "api": "wav_analysis_pixel_batch -> host WaveletDecomposition -> "
                   "wav_synthesis_pixel_batch (numpy in/out, reference run_trial's timed pair; "
                   "wall clock, synchronous copies; every array the drop-in returns, the "
                   "sh_synthesis input map included, is a page-locked block of torch's caching "
                   "host allocator)"}


def workload_config(cfgname, bands, mode, ws, map_bytes):
    """The `config` dict of the JSON line; the reference arm prints the same."""
    cfg = CONFIGS[cfgname]
    L, B, real = cfg["L"], cfg["batch"], cfg["real"]
    return {
        "workload": f"{cfgname}: L={L} MW {'real' if real else 'complex'} x{B}, "
                    f"lambda={cfg['lam']:g}, J0={cfg['j0']}, "
                    f"{'multires' if cfg['multires'] else 'full-res'}",
        "L": L, "batch": B, "bands": [int(b) for b in bands],
        "parallelism": {"single": "single GPU", "replica": f"replicas x{ws}",
                        "shard": f"orders/rings sharded x{ws} (fused exchange over peer memory or "
                                 "NCCL P2P; scales <= 256 whole on one rank)"}[mode],
        "l2": f"inputs larger than L2 (map {map_bytes / 1e6:.0f} MB, working set > 1 GB)"
              if L >= 1024 else "small config (L2-resident)",
    }


def hbm_stages(cfg, bands, stages):
    """Achieved HBM bandwidth of the ring-FFT / theta stages: algorithmic bytes
    per round trip (stage_bytes) / the stage's CUDA-event time per round trip."""
    peak, src = hbm_peak_gbs()
    out = {"peak_gbs": peak, "peak_source": src}
    for name, nb in stage_bytes(cfg, bands).items():
        ms = stages.get(name, {}).get("ms_per_step", 0.0)
        gbs = nb / (ms * 1e-3) / 1e9 if ms else None
        out[name] = {"bytes_per_rt": nb, "ms_per_rt": ms, "gbs": gbs,
                     "frac": gbs / peak if gbs else None}
    return out


def oracle_parity(cfg, f0, x0, sht):
    """Checker (not timed): the bench input map (our MW synthesis of the seeded
    f_lm) against the CPU oracle's direct Legendre sums on the MW rings at
    sampled orders -- including m in [651, 830], which the reference zeroes at
    L = 2048 -- normwise over those orders; and our MW analysis of
    that map against the seeded f_lm (normwise)."""
    import torch

    from oracle import oracle as orc

    L, real = cfg["L"], cfg["real"]
    N = 2 * L - 1
    orders = sorted({0, 1, 17, L // 4, L // 2, L - 2, L - 1} | {m for m in (651, 700, 760, 830)
                                                              if m < L})
    G = orc.legendre_synth(f0[None], L, real, "mw", orders=np.array(orders, np.int32))[0]
    F = (np.fft.rfft(x0.real, axis=-1) if real else np.fft.fft(x0, axis=-1)) / N
    bins = sorted({b for m in orders for b in ({m} if real else {m, (N - m) % N})})
    ref = G[:-1, bins]
    worst = float(np.abs(F[:-1, bins] - ref).max() / np.abs(ref).max())
    back = sht.analysis(torch.from_numpy(x0[None].copy()).cuda())[0].cpu().numpy()
    flm_err = float(np.abs(back - f0).max() / np.abs(f0).max())
    return {"oracle_synth_rel_err": worst, "orders": orders,
            "flm_rel_err": flm_err,
            "note": "max|ours - oracle| / max|oracle| over the ring Fourier modes of the input "
                    "map at the sampled orders (+-m; MW rings, pole ring excluded); flm_rel_err: "
                    "our analysis of that map vs the seeded f_lm, normwise; bar 1e-10"}


def cpu_baseline(cfgname, args):
    try:
        from oracle import oracle as orc
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "round-trips/s", "error": f"oracle unavailable: {e}"}
    return orc.bench_sample(CONFIGS[cfgname], seconds=args.cpu_seconds)


def run_reference(args, cfgname):
    ws, rank, _ = dist_env()
    if rank != 0:
        return None
    from oracle import oracle as orc

    cfg = CONFIGS[cfgname]
    steps = []
    for _ in range(args.warmup):
        orc.bench_sample(cfg, seconds=args.cpu_seconds)
    for _ in range(args.steps):
        steps.append(orc.bench_sample(cfg, seconds=args.cpu_seconds))
    vals = [s["value"] for s in steps]
    v = float(np.mean(vals))
    s0 = steps[0]
    return {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "round-trips/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 / v if v else None, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfgname, orc.sd_bands(cfg["L"], cfg["lam"], cfg["j0"],
                                                        cfg["multires"]),
                                  "single" if ws == 1 else (args.mode or "shard"), ws,
                                  cfg["batch"] * cfg["L"] * (2 * cfg["L"] - 1)
                                  * (8 if cfg["real"] else 16)),
        "cpu_baseline": {"value": v, "unit": "round-trips/s", "cores": s0["cores"],
                         "kind": s0["kind"], "coverage": s0["coverage"], "sample": s0["sample"]},
        "e2e": {"value": v, "unit": "round-trips/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="replay the round trip from a CUDA graph (auto: on, single/replica mode)")
    ap.add_argument("--exchange", choices=["peer", "nccl"], default="peer",
                    help="shard mode: fused exchange over peer memory (kernels store into the "
                         "owners' buffers) or grouped NCCL P2P messages")
    ap.add_argument("--mode", choices=["single", "shard", "replica"], default=None,
                    help="N=1: single; N>1 default shard (one map split by orders/rings, "
                         "strong scaling) or replica (independent maps, weak scaling)")
    args = ap.parse_args()
    # stdout carries exactly one JSON line: everything else written to fd 1 by
    # libraries (NCCL's version banner, torch) goes to stderr
    json_out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    rec = run_reference(args, args.config) if args.impl == "reference" else run_ours(args, args.config)
    if rec is not None:
        print(json.dumps(rec), file=json_out, flush=True)


if __name__ == "__main__":
    main()
