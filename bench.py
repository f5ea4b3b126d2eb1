"""Benchmark: ms per 8192-chirp 30 m x 30 m BP image and pixel.chirp updates/s on N B200s.

Contract (one JSON line from rank 0):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]
Under torchrun (N > 1) every rank runs one process per GPU; the image rows are sharded
across ranks (pixel-tile sharding) and assembled with an NCCL all_gather over NVLink,
the north star's multi-GPU design.  A step = range compression of all chirps
(sar_range_compress) + back-projection of this rank's rows (sar_backproject)
[+ all_gather_into_tensor when N > 1], inputs resident in HBM.

``--impl reference`` times the fp64 CPU oracle (oracle/) on the host cores, the
reference arm of this tier; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms per 8192-chirp 30×30 m BP image; pixel·chirp updates/s at 1/2/4/8 B200"
UNIT = "px·chirp·rx updates/s"
STREAM_METRIC = "ms per 8192-chirp streaming frame; image pixel·chirp updates/s"
WORKLOADS = {
    "C3": "C3: 8192 chirps x 512 samples, 1 RX, curved non-equidistant track (R = 20 m, 6->9 m/s), "
          "30 m x 30 m grid at 1 cm (3000 x 3000 px), Fig.1-style scene + 96 isolated points, AWGN 0.05",
    "C2": "C2: 8192 chirps x 512 samples, 1 RX, straight 8 m/s track, 30 m x 12 m at 1 cm (3000 x 1200 px)",
    "C0": "C0: paper grid 1201 x 1201 px at 2.5 cm over 30 m x 30 m, 8192 chirps, 1 RX (C2 track)",
    "C4": "C4: 8192 chirps x 4 RX (bistatic MIMO), 30 m x 30 m at 5 mm (6000 x 6000 px)",
    "C6": "C6: the paper's measurement, 1024 chirps x 8 RX (bistatic) = 8192 aperture samples, slow straight "
          "pass (0.75 m/s), paper grid 1201 x 1201 px at 2.5 cm over 30 m x 30 m",
    "C6p": "C6p (Measure E): C6 data on the polar grid of the recipe (factor 2.5, aperture 8.2 cm): 520 ranges "
           "x 315 bearings = 163,800 px (11.4 % of 1201^2), + bilinear resampling onto the 1201^2 grid",
}


# The paper's own numbers for the same workload (Table 2; GTX 1080 Ti, BP kernel time):
# context, not the target -- another machine.
PAPER_UPD_S = {
    "C6": (4.11e10, "paper Table 2 row 6 (P:L275-277): 1201^2 px x 1024 x 8 RX in 287.3 ms BP, GTX 1080 Ti"),
    "C6p": (8.72e10, "paper Table 2 row 8 (P:L284-286): 165,061 px x 1024 x 8 RX in 15.5 ms BP, GTX 1080 Ti"),
}


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - reported in the JSON line
            self.err = repr(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                r = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- helpers
def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def _alu_peak_upd_s(n_sm: int, mhz: float) -> float:
    """SFU roofline of the BP update: 3 MUFU-class ops (1 rsqrt, 1 sin, 1 cos) per update,
    16 MUFU results/clk/SM."""
    return n_sm * 16.0 * mhz * 1e6 / 3.0


def _traffic_from_profiles(cfg: str):
    p = os.path.join(ROOT, "profiles", "bp_dram_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(cfg)
    except Exception:
        return None


def _setup(cfg: str, device):
    import torch

    import sarsim

    scn = sarsim.make_config(cfg)
    raw = sarsim.simulate_raw(scn, device=str(device))
    return scn, raw


# ----------------------------------------------------------------------------- oracle arm
def _oracle_sample(scn, raw_np, target_s: float, nthreads: int = 0):
    """Time the oracle (as it stands) on a bounded sample: range compression of every
    chirp + BP of a strided pixel subset sized for about ``target_s`` seconds."""
    import numpy as np

    import oracle

    r = scn.radar
    g = scn.grid
    t0 = time.perf_counter()
    prof = oracle.range_compress(raw_np, r.fft_len, r.range_window, scn.wsar, nthreads=nthreads)
    t_rc = time.perf_counter() - t0
    # calibrate with growing probes (each call also pays the wrapper's profile copy), then
    # size the sample for about target_s seconds
    rng = np.random.default_rng(0)
    n_probe, t_probe = 256, 0.0
    while True:
        probe = g.pixel_list(np.stack([rng.integers(0, g.ny, n_probe), rng.integers(0, g.nx, n_probe)], 1))
        t0 = time.perf_counter()
        oracle.backproject(prof, 0, r, scn.tx, scn.rx, probe, nthreads=nthreads)
        t_probe = time.perf_counter() - t0
        if t_probe > 0.1 * target_s or n_probe >= g.nx * g.ny:
            break
        n_probe *= 4
    n_pix = int(max(64, min(g.nx * g.ny, n_probe * target_s / max(t_probe, 1e-4))))
    idx = np.stack([rng.integers(0, g.ny, n_pix), rng.integers(0, g.nx, n_pix)], 1)
    t0 = time.perf_counter()
    oracle.backproject(prof, 0, r, scn.tx, scn.rx, g.pixel_list(idx), nthreads=nthreads)
    t_bp = time.perf_counter() - t0
    full_pix = g.nx * g.ny
    est_image_s = t_rc + t_bp * full_pix / n_pix
    return {"t_rc_s": t_rc, "t_bp_s": t_bp, "n_pix": n_pix, "est_image_s": est_image_s,
            "value": scn.updates / est_image_s}


def run_reference(args):
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    import numpy as np
    import torch

    import sarsim

    cores = os.cpu_count() or 1
    scn = sarsim.make_config(args.config)
    raw = sarsim.simulate_raw(scn, device="cuda:0" if torch.cuda.is_available() else "cpu").cpu().numpy()
    per_step = []
    for s in range(args.warmup + args.steps):
        res = _oracle_sample(scn, raw, target_s=args.ref_step_s)
        if s >= args.warmup:
            per_step.append(res)
    est = statistics.median(r["est_image_s"] for r in per_step)
    value = scn.updates / est
    wall = sum(r["t_rc_s"] + r["t_bp_s"] for r in per_step) / len(per_step)
    sample = (f"per step: oracle range compression of all {scn.n_chirps * scn.n_rx} rows + oracle BP of "
              f"{per_step[0]['n_pix']} random pixels x {scn.n_chirps} chirps x {scn.n_rx} RX; "
              f"full-image time (ms_per_step) extrapolated per pixel from that sample")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": est * 1e3,
        "extrapolated": True, "sample_pixels": per_step[0]["n_pix"], "sample_fraction": per_step[0]["n_pix"] / scn.grid.nx / scn.grid.ny,
        "sample_wall_ms_per_step": wall * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, scn),
        "parallelism": f"fp64 CPU oracle, {cores} host threads (rank 0)",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "per_core": value / cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


# ----------------------------------------------------------------------------- our arm
def config_dict(args, scn):
    """The workload of the line: identical in both arms (the driver compares them)."""
    r = scn.radar
    return {"workload": WORKLOADS[args.config], "config": args.config, "pixels": scn.grid.nx * scn.grid.ny,
            "chirps": scn.n_chirps, "n_rx": scn.n_rx, "samples": r.n_samples, "fft_len": r.fft_len,
            "updates": scn.updates, "l2": L2_NOTE}


L2_NOTE = "256 MB buffer written between timed steps (outside the event span)"


def gather_summary(world, legs, check):
    """N > 1: the gather legs of the same run.  ``legs`` maps "fused" / "publish" / "nccl" to
    {"ms": per-step ms (max over ranks), "bp_ms": per-rank BP ms list, "collective_ms": per-rank
    ms of the collective / barrier after the BP} or None when the leg did not run."""
    out = {"world": world, "headline": None}
    for name in ("fused", "publish", "nccl"):
        leg = legs.get(name)
        out[f"{name}_ms"] = None if leg is None else leg["ms"]
        out[f"{name}_bp_ms_per_rank"] = None if leg is None else leg["bp_ms"]
        out[f"{name}_collective_ms_per_rank"] = None if leg is None else leg["collective_ms"]
        out[f"{name}_check"] = check.get(name)
    ok = [n for n in ("fused", "publish", "nccl") if legs.get(n) is not None and (check.get(n) or {}).get("ok")]
    if ok:
        out["headline"] = min(ok, key=lambda n: legs[n]["ms"])
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2306_09784_b200 import sar
    from paper_2306_09784_b200.dist import gather_rows, row_partition, tile_partition, tile_row_partition

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    elif args.all_legs:   # check run on one GPU: a one-rank group, both gather legs and their checks
        dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1, device_id=dev)
    dist_on = world > 1 or args.all_legs
    sar.load()

    scn, raw = _setup(args.config, dev)
    g = scn.grid
    lo, hi = scn.antenna_box(1e-3)
    plan = sar.Plan(scn.radar, g, scn.n_chirps, scn.n_rx, (lo, hi), device=local)
    tiles_x, tiles_y = plan.tiles
    ty = plan.info.tile_y
    # fused leg: a balanced block of absolute tiles per rank (+-1 tile); NCCL leg: whole tile rows
    t0, nt = tile_partition(tiles_x * tiles_y, world, rank)
    parts = [tile_row_partition(tiles_y, ty, g.ny, world, r) for r in range(world)]
    row0, nrow = parts[rank]
    tx = torch.as_tensor(scn.tx, device=dev)
    rx = None if scn.rx is None else torch.as_tensor(scn.rx, device=dev).contiguous()
    wsar = torch.as_tensor(scn.wsar, device=dev)
    prof = plan.empty_profiles()
    per = max(n for _, n in parts)
    local_buf = plan.empty_image(per)   # a block of `per` rows: the NCCL leg gathers equal chunks
    local_img = local_buf[:nrow]
    full_img = torch.empty((per * world, g.nx), dtype=torch.complex64, device=dev) if dist_on else local_img
    fused, fused_err = None, None
    if dist_on and args.gather in ("auto", "fused", "publish", "multicast"):
        from paper_2306_09784_b200.dist import FusedRowGather

        try:
            fused = FusedRowGather(g.ny, g.nx, dev, prefer_multicast=args.gather == "multicast")
        except Exception as e:  # no symmetric memory on this system: the NCCL leg alone
            fused_err = repr(e)[:200]
    # publish leg (SAR_SCATTER_PUBLISH): plain BP of the rank's tile block into its own symmetric
    # image, then one copy of the finished tiles to the peers' images
    pub_ptrs = fused.publish_ptrs(rank) if fused is not None and args.gather in ("auto", "publish") else None
    p0, pn = t0, nt
    polar = plan.polar
    if polar:   # Measure E: the polar image is resampled onto the Cartesian C0 grid in the step
        import sarsim

        cart = sarsim.make_config("C0", n_chirps=1).grid
        cart_img = torch.empty((cart.ny, cart.nx), dtype=torch.complex64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # 256 MB > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]

    def step_fused():
        plan.range_compress(raw, wsar, out=prof, stream=stream)
        ev[1].record(stream)
        plan.backproject_scatter_tiles(prof, tx, fused.ptrs, t0, nt, rx, multicast=fused.multicast, stream=stream)
        ev[2].record(stream)
        fused.barrier()
        if polar:
            sar.polar_to_cartesian(g, fused.image, cart, out=cart_img, stream=stream)

    def step_publish():
        plan.range_compress(raw, wsar, out=prof, stream=stream)
        ev[1].record(stream)
        plan.backproject_scatter_tiles(prof, tx, pub_ptrs, p0, pn, rx, publish=True, stream=stream)
        ev[2].record(stream)
        fused.barrier()
        if polar:
            sar.polar_to_cartesian(g, fused.image, cart, out=cart_img, stream=stream)

    def step_nccl():
        plan.range_compress(raw, wsar, out=prof, stream=stream)
        ev[1].record(stream)
        plan.backproject(prof, tx, rx, row0=row0, nrow=nrow, out=local_img, stream=stream)
        ev[2].record(stream)
        if dist_on:
            # equal chunks of `per` rows (a short last tile-row block carries padding rows)
            dist.all_gather_into_tensor(torch.view_as_real(full_img).view(-1), torch.view_as_real(local_buf).view(-1))
        if polar:
            sar.polar_to_cartesian(g, image_of_nccl(), cart, out=cart_img, stream=stream)

    def image_of_nccl():
        if not dist_on:
            return full_img
        if all(n == per for _, n in parts):
            return full_img[: g.ny]
        return torch.cat([full_img[r * per: r * per + n] for r, (_, n) in enumerate(parts)])

    def timed(step):
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        step_ms, bp_ms, rc_ms, coll_ms = [], [], [], []
        l0 = plan.launches
        if dist_on:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            for _ in range(args.steps):
                flush.zero_()
                ev[0].record(stream)
                step()
                ev[3].record(stream)
                ev[3].synchronize()
                step_ms.append(ev[0].elapsed_time(ev[3]))
                rc_ms.append(ev[0].elapsed_time(ev[1]))
                bp_ms.append(ev[1].elapsed_time(ev[2]))
                coll_ms.append(ev[2].elapsed_time(ev[3]))
        torch.cuda.synchronize()
        if dist_on:
            dist.barrier()
        mine = torch.tensor([sum(step_ms), sum(bp_ms), sum(rc_ms), sum(coll_ms)], dtype=torch.float64, device=dev)
        allr = [torch.zeros_like(mine) for _ in range(world)]
        if dist_on:
            dist.all_gather(allr, mine)
        else:
            allr = [mine]
        allr = torch.stack(allr).cpu() / args.steps
        return {"ms": float(allr[:, 0].max()), "bp_ms": [float(x) for x in allr[:, 1]],
                "rc_ms": [float(x) for x in allr[:, 2]], "collective_ms": [float(x) for x in allr[:, 3]],
                "launches": plan.launches - l0, "clocks": clk.summary(), "bp_mine_ms": sum(bp_ms) / len(bp_ms)}

    # ---------------- measured load balance (N > 1, outside the timed regions): tile costs depend on
    # the geometry (near-field tiles, derived-leg series terms), so equal tile counts are not equal
    # work.  Each rank times its BP block in a warm-up step, the blocks are re-cut on the measured
    # cost (dist.rebalance), twice; both legs, each on its own block kind.
    balance = {}
    if dist_on and not args.equal_blocks:   # (a one-rank --all-legs run exercises the same path)
        from paper_2306_09784_b200.dist import rebalance

        def measured(step):
            step()
            step()
            ev[2].synchronize()
            t = torch.tensor([ev[1].elapsed_time(ev[2])], dtype=torch.float64, device=dev)
            allt = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(allt, t)
            return [float(x) for x in allt]

        if fused is not None and args.gather != "publish":
            tblocks = [tile_partition(tiles_x * tiles_y, world, r) for r in range(world)]
            hist = []
            for _ in range(2):
                times = measured(step_fused)
                hist.append(times)
                tblocks = [rebalance(tblocks, times, world, r) for r in range(world)]
                t0, nt = tblocks[rank]
            balance["fused"] = {"bp_ms_per_rank_before": hist[0], "bp_ms_per_rank_iter1": hist[1],
                                "tiles_per_rank": [n for _, n in tblocks]}
        if pub_ptrs is not None:
            pblocks = [tile_partition(tiles_x * tiles_y, world, r) for r in range(world)]
            hist = []
            for _ in range(2):
                times = measured(step_publish)
                hist.append(times)
                pblocks = [rebalance(pblocks, times, world, r) for r in range(world)]
                p0, pn = pblocks[rank]
            balance["publish"] = {"bp_ms_per_rank_before": hist[0], "bp_ms_per_rank_iter1": hist[1],
                                  "tiles_per_rank": [n for _, n in pblocks]}
        rblocks = [row_partition(tiles_y, world, r) for r in range(world)]   # = tile_row_partition's blocks
        hist = []
        for _ in range(2):
            times = measured(step_nccl)
            hist.append(times)
            rblocks = [rebalance(rblocks, times, world, r) for r in range(world)]
            parts = [(min(g.ny, a * ty), min(g.ny, (a + n) * ty) - min(g.ny, a * ty)) for a, n in rblocks]
            row0, nrow = parts[rank]
            per = max(n for _, n in parts)
            local_buf = plan.empty_image(per)
            local_img = local_buf[:nrow]
            full_img = torch.empty((per * world, g.nx), dtype=torch.complex64, device=dev)
        balance["nccl"] = {"bp_ms_per_rank_before": hist[0], "bp_ms_per_rank_iter1": hist[1],
                           "tile_rows_per_rank": [n for _, n in rblocks]}

    legs, check, snaps = {}, {}, {}
    if fused is not None and args.gather != "publish":
        legs["fused"] = timed(step_fused)
        if dist_on:
            snaps["fused"] = fused.image.clone()   # (the publish leg reuses the symmetric image)
    if pub_ptrs is not None:
        legs["publish"] = timed(step_publish)
        if dist_on:
            snaps["publish"] = fused.image.clone()
    legs["nccl"] = timed(step_nccl)
    # ---------------- outside the timed regions: every leg's image against this plan's 1-GPU image
    # (every pixel is computed in its absolute tile: equal up to the fp32 order of chirp-chunk sums)
    # (the DESIGN's "<= 1e-6" is the measured rank-partition case; the check allows T11's 1e-5)
    if dist_on:
        ref = plan.backproject(prof, tx, rx, stream=stream)
        torch.cuda.synchronize()
        scale = ref.abs().max().clamp_min(1e-30)
        imgs = {"nccl": image_of_nccl(), **snaps}
        for name, im in imgs.items():
            rel = float((im - ref).abs().max() / scale)
            # T11: 1e-5, the fp32 order of chirp-chunk sums (legs split their chirps
            # differently; every pixel's anchor and derived-leg grouping are the same)
            check[name] = {"max_rel_diff_to_1gpu_image": rel, "equal": bool(torch.equal(im, ref)), "ok": rel <= 1e-5}
        flags = torch.tensor([0 if c["ok"] else 1 for c in check.values()], device=dev)
        dist.all_reduce(flags, op=dist.ReduceOp.MAX)   # every rank agrees on the verdict
        for name, bad in zip(check, flags.tolist()):
            check[name]["ok"] = check[name]["ok"] and not bad
        del ref
    else:
        check["nccl"] = {"ok": True}
    gather = gather_summary(world, legs, check) if dist_on else None
    if gather is not None and balance:
        gather["balance"] = balance
    head = "nccl" if not dist_on else gather["headline"]
    if head is None:   # no leg produced the 1-GPU image: report the failure, no number
        if rank == 0:
            emit({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world, "invalid":
                  "no gather leg reproduced the 1-GPU image", "gather": gather, "config": config_dict(args, scn)})
        plan.close()
        if dist_on:
            dist.destroy_process_group()
        return 1
    leg = legs[head]
    ms_per_step = leg["ms"]
    value = scn.updates / (ms_per_step * 1e-3)

    # ---------------- roofline of the dominant kernel (bp_kernel), this rank's launches
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    peaks = _peaks()
    clocks = leg["clocks"]
    max_mhz = float(peaks.get("sm_max_mhz", clocks.get("sm_max_mhz") or 1965.0))
    if head in ("fused", "publish"):
        # pixels of the rank's tiles (ragged last tile column / row clipped to the grid)
        b0, bn = (t0, nt) if head == "fused" else (p0, pn)
        ntx = [min(32, g.nx - 32 * (t % tiles_x)) for t in range(b0, b0 + bn)]
        nty = [min(ty, g.ny - ty * (t // tiles_x)) for t in range(b0, b0 + bn)]
        bp_px = sum(a * b for a, b in zip(ntx, nty))
    else:
        bp_px = nrow * g.nx
    bp_upd = bp_px * scn.n_chirps * scn.n_rx
    bp_avg_s = leg["bp_mine_ms"] * 1e-3
    achieved = bp_upd / bp_avg_s
    peak = _alu_peak_upd_s(n_sm, max_mhz)
    roofline = {
        "bound": "alu", "achieved": achieved, "peak": peak, "unit": "upd/s", "frac": achieved / peak,
        "traffic": _traffic_from_profiles(args.config),
        "kernel": "bp_kernel", "peak_basis": f"SFU: {n_sm} SM x 16 MUFU/clk x {max_mhz:.0f} MHz / 3 MUFU per update",
        "frac_at_measured_clock": (achieved / _alu_peak_upd_s(n_sm, clocks["sm_mhz"])) if clocks.get("sm_mhz") else None,
        "bp_ms": bp_avg_s * 1e3, "rc_ms": leg["rc_ms"][rank],
    }

    # ---------------- end to end through the C ABI with host buffers (sar_form_image)
    raw_h = raw.cpu().pin_memory()
    tx_h = torch.as_tensor(scn.tx).contiguous().pin_memory()
    rx_h = None if scn.rx is None else torch.as_tensor(scn.rx).contiguous().pin_memory()
    wsar_h = torch.as_tensor(scn.wsar).pin_memory()
    img_h = torch.empty((nrow, g.nx), dtype=torch.complex64).pin_memory()
    e2e_steps = max(1, min(args.steps, 5))
    for _ in range(2):
        plan.form_image(raw_h, tx_h, rx_h, wsar_h, row0=row0, nrow=nrow, out_h=img_h, stream=stream)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_ms = 0.0
    for _ in range(e2e_steps):
        flush.zero_()
        e0.record(stream)
        plan.form_image(raw_h, tx_h, rx_h, wsar_h, row0=row0, nrow=nrow, out_h=img_h, stream=stream, sync=False)
        e1.record(stream)
        e1.synchronize()
        e2e_ms += e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t[0])
    e2e_ms /= e2e_steps
    h2d = raw_h.numel() * 4 + tx_h.numel() * 8 + wsar_h.numel() * 4 + (0 if rx_h is None else rx_h.numel() * 8)
    d2h = img_h.numel() * 8

    # ---------------- "Load" as in the paper's Table 2 (Measure C): pinned H2D of the raw
    # samples and poses on its own (inside e2e it overlaps nothing: sar_form_image's range
    # compression reads the pinned raw rows in place)
    raw_d, tx_d = torch.empty_like(raw), torch.empty_like(tx)
    load_ms = 0.0
    for i in range(e2e_steps + 1):
        e0.record(stream)
        with torch.cuda.stream(stream):
            raw_d.copy_(raw_h.view_as(raw_d), non_blocking=True)
            tx_d.copy_(tx_h, non_blocking=True)
        e1.record(stream)
        e1.synchronize()
        if i:
            load_ms += e0.elapsed_time(e1)
    load_ms /= e2e_steps
    del raw_d, tx_d

    # ---------------- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res = _oracle_sample(scn, raw.cpu().numpy(), target_s=args.cpu_s)
        cpu = {"value": res["value"], "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
               "per_core": res["value"] / (os.cpu_count() or 1),
               "sample": f"oracle range compression of all {scn.n_chirps * scn.n_rx} rows "
                         f"({res['t_rc_s']:.2f} s) + oracle BP of {res['n_pix']} random pixels x all chirps "
                         f"({res['t_bp_s']:.2f} s), full image extrapolated to {res['est_image_s']:.1f} s"}

    if rank == 0:
        if head == "nccl" and world == 1:
            par, step_txt = "pixel tiles x1", "sar_range_compress(all chirps) + sar_backproject(all rows)"
        elif head == "fused":
            par = (f"pixel tiles x{world} (balanced tile blocks) + gather fused into the BP epilogue "
                   f"({'multimem.st' if fused.multicast else 'P2P stores'}, symmetric memory)")
            step_txt = ("sar_range_compress(all chirps) + sar_backproject_scatter_tiles(rank tiles -> every "
                        "rank's image) + symmetric-memory barrier")
        elif head == "publish":
            par = (f"pixel tiles x{world} (balanced tile blocks) + BP into the own symmetric-memory image, "
                   f"then one copy of the finished tiles to every peer (P2P stores)")
            step_txt = ("sar_range_compress(all chirps) + sar_backproject_scatter_tiles(SAR_SCATTER_PUBLISH: rank "
                        "tiles -> own image -> every rank's image) + symmetric-memory barrier")
        else:
            par = f"pixel tiles x{world} (blocks of whole tile rows) + NCCL all_gather_into_tensor"
            step_txt = "sar_range_compress(all chirps) + sar_backproject(rank tile rows) + all_gather_into_tensor"
        if polar:
            step_txt += " + sar_polar_to_cartesian"
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": (value / PAPER_UPD_S[args.config][0]) if args.config in PAPER_UPD_S else None,
            "baseline_note": PAPER_UPD_S[args.config][1] if args.config in PAPER_UPD_S else None,
            "dtype": "f32", "data": "synthetic",
            "config": config_dict(args, scn),
            "parallelism": par, "step": step_txt, "n_bins": plan.n_bins,
            "gather": gather, "fused_gather_error": fused_err,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": scn.updates / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_image": e2e_ms,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "load_ms": load_ms, "load_note": "pinned H2D of raw samples + poses alone (Table 2 'Load')",
                    "api": "sar_form_image (C ABI, pinned host buffers: H2D poses, rc reading the pinned raw "
                           "samples in place, bp in 4 bands of tile rows with each band's D2H copy overlapping "
                           "the next band)"
                           + ("" if world == 1 else "; each rank its tile-row block")},
            "gpu_launches": leg["launches"],
            "clocks": clocks,
        }
        emit(line)
    plan.close()
    if dist_on:
        dist.destroy_process_group()
    return 0


def run_stream(args):
    """C5: streaming sliding-window frames (8192-chirp apertures, 1024-chirp hop), one image per
    frame, chirps sharded across ranks and summed with an NCCL reduce to rank 0.  A step is one
    frame: range compression of this rank's chirps of the frame + back-projection of those chirps
    over the frame grid + reduce.  Reports per-frame latency against the real-time budget
    N_m T_P0 = 1024 x 106.7 us = 109.3 ms per hop."""
    import torch
    import torch.distributed as dist

    import sarsim
    from paper_2306_09784_b200 import sar
    from paper_2306_09784_b200.dist import chirp_partition, reduce_partials

    world, rank, local = _env_int("WORLD_SIZE", 1), _env_int("RANK", 0), _env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    sar.load()
    scn = sarsim.make_config("C5")
    frames = sarsim.c5_frames(scn)
    raw = sarsim.simulate_raw(scn, device=str(dev))
    tx = torch.as_tensor(scn.tx, device=dev)
    wsar = torch.as_tensor(scn.wsar, device=dev)
    lo, hi = scn.antenna_box(1e-3)
    plans = [sar.Plan(scn.radar, g, scn.n_chirps, 1, (lo, hi), device=local) for _, g in frames]
    nb_max = max(p.n_bins for p in plans)
    prof_buf = torch.empty(scn.n_chirps * nb_max, dtype=torch.complex64, device=dev)
    g0 = frames[0][1]
    img = torch.empty((g0.ny, g0.nx), dtype=torch.complex64, device=dev)
    stream = torch.cuda.current_stream(dev)
    c_lo, c_n = chirp_partition(8192, world, rank)
    # N > 1: the chirp-shard reduction fused into the BP epilogue (P2P red.add into rank 0's
    # symmetric-memory image; --gather nccl keeps the separate reduce)
    fused = None
    if world > 1 and args.gather in ("fused", "multicast") and args.config != "C5i":
        from paper_2306_09784_b200.dist import FusedRowGather

        try:
            fused = FusedRowGather(g0.ny, g0.nx, dev, prefer_multicast=False)
        except Exception as e:
            print(f"bench: fused reduce unavailable ({e!r}); using NCCL", file=sys.stderr)

    incremental = args.config == "C5i"
    if incremental:
        # NEXT-2: world-fixed grid (the C2 grid), one partial image per 1024-chirp hop in a ring
        # of 8; a frame = back-projection of the newest hop + sum of the ring
        g0 = scn.grid
        plans.append(sar.Plan(scn.radar, g0, scn.n_chirps, 1, (lo, hi), device=local))
        ring = torch.zeros((8, g0.ny, g0.nx), dtype=torch.complex64, device=dev)
        iplan = plans[-1]
        iprof = iplan.empty_profiles()
        h_lo, h_n = chirp_partition(1024, world, rank)
        img = torch.empty((g0.ny, g0.nx), dtype=torch.complex64, device=dev)

    def frame(f):
        if incremental:
            h = f % (scn.n_chirps // 1024)
            iplan.range_compress(raw, wsar, chirp0=h * 1024 + h_lo, nchirp=h_n, out=iprof, stream=stream)
            iplan.backproject(iprof, tx, chirp0=h * 1024 + h_lo, nchirp=h_n, out=ring[h % 8], stream=stream)
            if world > 1:
                reduce_partials(ring[h % 8], dst=0)
            sar.image_sum(ring, out=img, stream=stream)
            return
        c0, _ = frames[f % len(frames)]
        plan = plans[f % len(frames)]
        prof = prof_buf[: scn.n_chirps * plan.n_bins].view(scn.n_chirps, 1, plan.n_bins)
        plan.range_compress(raw, wsar, chirp0=c0 + c_lo, nchirp=c_n, out=prof, stream=stream)
        if fused is not None:
            if rank == 0:
                fused.image.zero_()
            fused.barrier()
            plan.backproject_scatter(prof, tx, fused.root_ptrs(0), chirp0=c0 + c_lo, nchirp=c_n, add=True,
                                     stream=stream)
            fused.barrier()
            return
        plan.backproject(prof, tx, chirp0=c0 + c_lo, nchirp=c_n, out=img, stream=stream)
        if world > 1:
            reduce_partials(img, dst=0)

    for f in range(args.warmup):
        frame(f)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    l0 = sum(p.launches for p in plans)
    with ClockSampler(local) as clk:
        for f in range(args.steps):
            e0.record(stream)
            frame(f)
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
    launches = sum(p.launches for p in plans) - l0
    tot = torch.tensor([sum(ms), max(ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_frame = float(tot[0]) / args.steps
    upd = g0.nx * g0.ny * 8192          # updates of the frame's 8192-chirp image
    if incremental:
        workload = ("C5i (NEXT-2 incremental): world-fixed 30 m x 12 m grid at 1 cm, 8 partial images of "
                    "1024-chirp hops in a ring; a frame = BP of the newest hop + ring sum")
        step = "one frame: sar_range_compress + sar_backproject of one hop (+ reduce) + sar_image_sum"
    else:
        workload = ("C5: 16 frames of 8192 chirps, 1024-chirp hop, straight 8 m/s track, "
                    "30 m x 12 m grid at 1 cm re-centred per frame")
        step = "one frame: sar_range_compress + sar_backproject of this rank's chirps (+ reduce)"
    if rank == 0:
        emit({
            "metric": STREAM_METRIC,
            "value": upd / (ms_frame * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_frame, "max_frame_ms": float(tot[1]),
            "realtime_budget_ms": 1024 * scn.radar.pri_s * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload, "config": args.config,
                       "parallelism": f"chirps x{world}" + (
                           "" if world == 1 else
                           " + reduction fused into the BP epilogue (P2P red.add, symmetric memory)" if fused is not None
                           else " + NCCL reduce"),
                       "step": step},
            "gpu_launches": launches, "clocks": clk.summary(),
        })
    for p in plans:
        p.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


_OUT = None   # the process's real stdout once main() has claimed it (see _claim_stdout)


def _claim_stdout():
    """The JSON line is the only stdout line: keep the real stdout on a private descriptor and point
    descriptor 1 at stderr, so that anything else a library prints there (NCCL's version banner, which
    rank 0 of a process group prints on stdout whatever NCCL_DEBUG says) cannot precede or split it."""
    global _OUT
    if _OUT is None:
        sys.stdout.flush()
        _OUT = os.fdopen(os.dup(1), "w", buffering=1)
        os.dup2(2, 1)
    return _OUT


def emit(obj):
    print(json.dumps(obj), file=_OUT or sys.stdout, flush=True)


def main(argv=None):
    # the JSON line is the only stdout line: NCCL's version banner (NCCL_DEBUG=VERSION) would precede it
    if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
        os.environ["NCCL_DEBUG"] = "WARN"
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=sorted(WORKLOADS) + ["C5", "C5i"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-s", type=float, default=12.0, help="seconds of oracle BP for cpu_baseline")
    ap.add_argument("--ref-step-s", type=float, default=4.0, help="seconds of oracle BP per reference step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--equal-blocks", action="store_true",
                    help="N > 1: equal tile (row) counts per rank, no measured load balance")
    ap.add_argument("--all-legs", action="store_true",
                    help="N = 1 check run: a one-rank process group, both gather legs timed and checked")
    ap.add_argument("--gather", default="auto", choices=["auto", "fused", "publish", "multicast", "nccl"],
                    help="N > 1, image configs: besides the NCCL all_gather leg (always timed), time the gather "
                         "fused into the BP epilogue (auto/fused: P2P stores, multicast: multimem.st to the "
                         "NVSwitch multicast address; symmetric memory) and the publish leg (auto/publish: BP into "
                         "the own image, then one copy of the tiles to the peers); nccl: the NCCL leg only.  C5: the "
                         "chirp-shard reduction is an NCCL reduce unless fused/multicast (P2P red.add)")
    args = ap.parse_args(argv)
    _claim_stdout()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        if args.config in ("C5", "C5i"):
            raise SystemExit("--impl reference supports the image configs (C0-C4)")
        return run_reference(args)   # rank 0 alone (any launch); other ranks exit 0
    world = _env_int("WORLD_SIZE", 1)
    if world != args.gpus:
        if "WORLD_SIZE" in os.environ or args.gpus < 1:
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
        return self_launch(args, argv)
    return run_stream(args) if args.config in ("C5", "C5i") else run_ours(args)


def self_launch(args, argv):
    """``bench.py --gpus N`` outside torchrun: start N ranks (one per GPU) with torchrun on this
    node; rank 0's JSON line is the output.  With fewer than N GPUs visible, one JSON line says so
    (no ranks sharing a GPU: their numbers would not be N-GPU numbers)."""
    import socket
    import subprocess

    try:
        import torch

        ngpu = torch.cuda.device_count()
    except Exception:
        ngpu = 0
    if ngpu < args.gpus:
        legs = {"fused": None, "publish": None, "nccl": None}
        emit({"metric": METRIC if args.config not in ("C5", "C5i") else STREAM_METRIC, "value": None,
              "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
              "unavailable": f"--gpus {args.gpus}: {ngpu} GPU(s) visible",
              "gather": gather_summary(args.gpus, legs, {})})
        return 0
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    argv = list(sys.argv[1:] if argv is None else argv)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]
    # the ranks write their JSON line to this process's real stdout (descriptor 1 points at stderr)
    return subprocess.call(cmd, stdout=_OUT)


if __name__ == "__main__":
    sys.exit(main())
