#!/usr/bin/env python
"""GaussianImage hot-path benchmark on B200 (driver contract).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (configs[1], "C2"): a Kodak-shaped 768x512 synthetic image fitted by
70,000 Gaussians (560K parameters, Table 1) with Adam.  A STEP is one
fit iteration of the whole hot path: project (+ per-tile key counts) ->
tile-bin (counting sort on the tile id + per-tile gid sort, no depth key) ->
fused forward (Eq. 7) + L2 loss + Appendix-A backward -> per-Gaussian
finalize fused with Adam (paper schedule).  The JSON line's `value` is
fit iterations/s over all ranks; `render_fps` (project + bin + render) and
`decode_fps` (RVQ/fp16/b-bit decode + project + bin + render, configs[4] at
70k records) are measured in the same run.  The L2 cache (126 MB) is flushed
with a 256 MB write before every timed step (the C2 working set is ~60 MB).

Multi-GPU (torchrun): each rank fits its own image (weak scaling, no
collective on the data path); per-image PSNR is all-gathered over NCCL at
the end; timings are the max over ranks.

--impl reference: the fp64 CPU oracle (oracle/), unmodified, timed on the
host cores for the same metric -- rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("render FPS + fit iters/s @768×512, 70k Gaussians; fraction of FP32/HBM "
          "roofline")
W_IMG, H_IMG, N_GAUSS = 768, 512, 70000
PAPER_FIT_ITS = 50000 / 106.59        # Table 1a, V100, Adan: 469.1 it/s
L2_FLUSH_BYTES = 256 << 20
# algorithmic FP32 work per (pixel, Gaussian) pair in the box:
#   forward  (Eq. 5 + 7, factored conic): 15 FLOP + 1 ex2
#   backward (App. A, 5-moment form)   : 34 FLOP + 1 ex2
FLOP_PER_PAIR_FUSED = 15 + 34
FLOP_PER_PAIR_RENDER = 15
FP32_LANES_PER_SM = 128
N_SM = 148


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--batch-images", type=int, default=-1,
                    help="images per launch for the extra batched measurement (0 = skip; "
                         "default: configs[3], 64 images sharded over the ranks)")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------ clocks
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(self.NAMES, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- reference
def run_reference(args):
    """The oracle, as it stands, on the host cores: C2 fit iterations."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synth
    from oracle import gio
    p = synth.init_params(1, N_GAUSS)
    tgt = synth.image(1, W_IMG, H_IMG)
    m = np.zeros_like(p)
    v = np.zeros_like(p)

    def it(step, p, m, v):
        _, loss, g = gio.loss_and_grads(p, tgt, mode=gio.TILED)
        po, mo, vo = gio.adam(p, g.astype(np.float32), m, v, step, gio.lr_at(step))
        return po.astype(np.float32), mo.astype(np.float32), vo.astype(np.float32), loss

    t0 = time.time()
    p, m, v, _ = it(1, p, m, v)
    est = time.time() - t0
    budget = 150.0
    warm = max(0, min(args.warmup, int(30.0 / max(est, 1e-3))))
    steps = max(1, min(args.steps, int(budget / max(est, 1e-3))))
    step = 2
    for _ in range(warm):
        p, m, v, _ = it(step, p, m, v)
        step += 1
    t0 = time.perf_counter()
    for _ in range(steps):
        p, m, v, loss = it(step, p, m, v)
        step += 1
    dt = time.perf_counter() - t0
    val = steps / dt
    cores = gio.num_threads()
    sample = (f"{steps} fp64 oracle fit iterations (tiled render + L2 + Appendix-A backward + "
              f"Adam) of C2 768x512 / 70k Gaussians")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "it/s",
            "n_gpus": args.gpus, "steps": args.steps, "steps_timed": steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * dt / steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C2: Kodak-shaped 768x512 synthetic image, 70k Gaussians, "
                                   "Adam fit step", "oracle_threads": cores},
            "cpu_baseline": {"value": val, "unit": "it/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": val, "unit": "it/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def cpu_baseline(seconds: float):
    import synth
    from oracle import gio
    p = synth.init_params(1, N_GAUSS)
    tgt = synth.image(1, W_IMG, H_IMG)
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    n = 0
    t0 = time.perf_counter()
    while True:
        _, loss, g = gio.loss_and_grads(p, tgt, mode=gio.TILED)
        po, mo, vo = gio.adam(p, g.astype(np.float32), m, v, n + 1, gio.lr_at(n + 1))
        p, m, v = po.astype(np.float32), mo.astype(np.float32), vo.astype(np.float32)
        n += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "it/s", "cores": gio.num_threads(), "kind": "oracle",
            "sample": f"{n} fp64 oracle fit iterations of C2 (768x512, 70k Gaussians, tiled "
                      f"render + L2 + backward + Adam) in {dt:.1f} s"}


# ------------------------------------------------------------------- ours
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import synth
    from paper_2403_08551_b200 import gi
    from paper_2403_08551_b200.dist import gather_psnr
    from paper_2403_08551_b200.pipeline import Fitter, Pipeline

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    gi.load()
    K, Wm = max(1, args.steps), max(3, args.warmup)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    seed = 1 + rank
    p_host = synth.init_params(seed, N_GAUSS)
    t_host = synth.image(seed, W_IMG, H_IMG)
    params = torch.from_numpy(p_host).to(dev).view(1, N_GAUSS, 8).contiguous()
    target = torch.from_numpy(t_host).to(dev).view(1, 3, H_IMG, W_IMG).contiguous()
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    clocks = Clocks(local)

    # ---------------- fit step (value) ----------------
    # Two graphs of one fused step: `plain` (what `value` times) and `staged`
    # (external event nodes at the stage boundaries, for the stage split and
    # the roofline kernel time).  Event nodes cost several us each inside a
    # graph, so they are kept out of the timed value.
    fit = Fitter(params.clone(), target)
    fit.step()
    torch.cuda.synchronize(dev)
    st = fit.check()
    if st != gi.GI_OK:
        raise RuntimeError(f"fit status {st}")
    n0 = gi.gi_launch_count()
    plain_g = fit.capture(1)
    launches_per_step = gi.gi_launch_count() - n0
    stage_ev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(6)]
    for e in stage_ev:
        e.record(stream)
    torch.cuda.synchronize(dev)
    staged_g = fit.capture(1, stage_events=stage_ev)
    for _ in range(Wm):
        plain_g.replay()
    torch.cuda.synchronize(dev)
    # pair count for the roofline at the state the timed steps start from
    probe = Pipeline(N_GAUSS, W_IMG, H_IMG, 1, device=dev)
    probe.project(fit.params)
    rec = probe.proj.view(-1, 12).cpu().numpy()
    bx, by = rec[:, 7].view(np.uint32), rec[:, 11].view(np.uint32)
    wx = (bx >> 16).astype(np.int64) - (bx & 0xffff).astype(np.int64) + 1
    wy = (by >> 16).astype(np.int64) - (by & 0xffff).astype(np.int64) + 1
    touched = probe.tiles_touched.cpu().numpy() > 0
    pairs = int(np.sum(np.where(touched, wx * wy, 0)))
    keys = int(probe.tiles_touched.cpu().numpy().astype(np.int64).sum())
    del probe

    s_ev = [torch.cuda.Event(enable_timing=True) for _ in range(max(K, 10))]
    e_ev = [torch.cuda.Event(enable_timing=True) for _ in range(max(K, 10))]
    barrier()
    clocks.start()
    for i in range(K):
        flush.zero_()
        s_ev[i].record(stream)
        plain_g.replay()
        e_ev[i].record(stream)
    barrier()
    fit_ms = sum(s_ev[i].elapsed_time(e_ev[i]) for i in range(K))
    fit_ms_max = max_over_ranks(fit_ms)
    fit_value = world * K / (fit_ms_max / 1000.0)
    # stage split (instrumented graph, same flush protocol)
    stage_ms = np.zeros(5)   # [empty], [empty], tile kernel, finalize+Adam+next projection, tail
    KS = min(K, 100)
    for i in range(KS):
        flush.zero_()
        staged_g.replay()
        torch.cuda.synchronize(dev)
        for j in range(5):
            stage_ms[j] += stage_ev[j].elapsed_time(stage_ev[j + 1])
    stage_ms /= KS
    st = fit.check()
    if st != gi.GI_OK:
        raise RuntimeError(f"fit status after timing {st}")

    # ---------------- render FPS (gi_render_frame: project+count -> bin -> render) --------
    pipe = Pipeline(N_GAUSS, W_IMG, H_IMG, 1, device=dev)
    rparams = params.clone()
    pipe.render_frame(rparams)
    torch.cuda.synchronize(dev)
    rs = torch.cuda.Stream(device=dev)
    rs.wait_stream(stream)
    rg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(rg, stream=rs):
        pipe.render_frame(rparams)
    stream.wait_stream(rs)
    for _ in range(Wm):
        rg.replay()
    barrier()
    for i in range(K):
        flush.zero_()
        s_ev[i].record(stream)
        rg.replay()
        e_ev[i].record(stream)
    barrier()
    r_ms = sum(s_ev[i].elapsed_time(e_ev[i]) for i in range(K))
    render_fps = world * K / (max_over_ranks(r_ms) / 1000.0)
    # render-kernel-only time (ABI gi_render on gi_bin output, events around it)
    pipe.project(rparams)
    pipe.bin()
    r_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    r_kernel_ms = 0.0
    for i in range(K):
        flush.zero_()
        r_ev[0].record(stream)
        pipe.raster()
        r_ev[1].record(stream)
        torch.cuda.synchronize(dev)
        r_kernel_ms += r_ev[0].elapsed_time(r_ev[1])
    r_kernel_ms /= K
    render_pairs = pairs_of(pipe, np)

    # ---------------- decode FPS (configs[4]): gi_decode_render_frame (decode fused into project) ----
    data, gamma, beta, books = synth.payload(seed, N_GAUSS)
    d_payload = torch.from_numpy(data).to(dev)
    d_books = torch.from_numpy(books).to(dev)
    dparams = torch.zeros(1, N_GAUSS, 8, dtype=torch.float32, device=dev)
    meta = gi.codec_meta(N_GAUSS, gamma, beta, d_books)
    dpipe = Pipeline(N_GAUSS, W_IMG, H_IMG, 1, device=dev)
    gi.gi_vq_decode(d_payload, meta, dparams)
    dpipe.render_frame(dparams, gi.GI_POS_NORMALIZED)
    torch.cuda.synchronize(dev)
    ds = torch.cuda.Stream(device=dev)
    ds.wait_stream(stream)
    dg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(dg, stream=ds):
        dpipe.decode_render_frame(d_payload, meta, dparams)
    stream.wait_stream(ds)
    for _ in range(Wm):
        dg.replay()
    barrier()
    for i in range(K):
        flush.zero_()
        s_ev[i].record(stream)
        dg.replay()
        e_ev[i].record(stream)
    barrier()
    d_ms = sum(s_ev[i].elapsed_time(e_ev[i]) for i in range(K))
    decode_fps = world * K / (max_over_ranks(d_ms) / 1000.0)
    # codec-realistic record counts (~0.3 / 0.6 bpp at 56-bit records)
    decode_small = {}
    for n_small in (2200, 4500):
        sdata, sg, sb, sbooks = synth.payload(seed, n_small)
        s_pay = torch.from_numpy(sdata).to(dev)
        s_books = torch.from_numpy(sbooks).to(dev)
        s_meta = gi.codec_meta(n_small, sg, sb, s_books)
        s_params = torch.zeros(1, n_small, 8, dtype=torch.float32, device=dev)
        s_pipe = Pipeline(n_small, W_IMG, H_IMG, 1, device=dev)
        s_pipe.decode_render_frame(s_pay, s_meta, s_params)
        torch.cuda.synchronize(dev)
        sgs = torch.cuda.Stream(device=dev)
        sgs.wait_stream(stream)
        sgr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(sgr, stream=sgs):
            s_pipe.decode_render_frame(s_pay, s_meta, s_params)
        stream.wait_stream(sgs)
        for _ in range(Wm):
            sgr.replay()
        barrier()
        for i in range(K):
            flush.zero_()
            s_ev[i].record(stream)
            sgr.replay()
            e_ev[i].record(stream)
        barrier()
        sms = sum(s_ev[i].elapsed_time(e_ev[i]) for i in range(K))
        decode_small[str(n_small)] = world * K / (max_over_ranks(sms) / 1000.0)
        del sgr, s_pipe

    # ---------------- Adan fit step (the paper's optimiser, NEXT-1) ----------------
    afit = Fitter(params.clone(), target, optimizer="adan")
    afit.step()
    torch.cuda.synchronize(dev)
    ag = afit.capture(1)
    for _ in range(Wm):
        ag.replay()
    barrier()
    for i in range(K):
        flush.zero_()
        s_ev[i].record(stream)
        ag.replay()
        e_ev[i].record(stream)
    barrier()
    adan_value = world * K / (max_over_ranks(sum(s_ev[i].elapsed_time(e_ev[i]) for i in range(K)))
                              / 1000.0)
    if afit.check() != gi.GI_OK:
        raise RuntimeError("adan fit status")
    del afit, ag

    # ---------------- the paper's training run: 50k steps (106.59 s on V100) ----
    # Adam (north_star) and Adan (the paper's), chained, CUDA graphs of 100 steps,
    # warm L2 as a real fit runs; device time (events), max over ranks; final PSNR
    full_fit = {}
    psnr_pipe = Pipeline(N_GAUSS, W_IMG, H_IMG, 1, device=dev)
    for opt in ("adam", "adan"):
        ffit = Fitter(params.clone(), target, optimizer=opt)
        ffit.step()
        torch.cuda.synchronize(dev)
        fg = ffit.capture(100)
        barrier()
        s_ev[0].record(stream)
        for _ in range(500):                  # 1 + 500 x 100 = 50,001 steps
            fg.replay()
        e_ev[0].record(stream)
        barrier()
        secs = max_over_ranks(s_ev[0].elapsed_time(e_ev[0])) / 1000.0
        img = psnr_pipe.render_frame(ffit.params)
        full_fit[opt] = {"steps": 50001, "seconds": secs,
                         "psnr_db": float(psnr_pipe.psnr(img, target)[0])}
        if ffit.check() != gi.GI_OK:
            raise RuntimeError("50k fit status")
        if opt == "adam":
            fitted = ffit.params.clone()
        del ffit, fg

    # ---------------- the fitted state (SURVEY d.1): render FPS of the cloud the
    # 50k-step fit produced, and configs[4] from it -- C5 payload built as the
    # survey's recipe: fp16 positions, l codes with gamma = (max - min)/63,
    # beta = min, colours by 5 K-means iterations per RVQ stage (gi_kmeans_step,
    # B = 8, M = 2), packed by gi_vq_encode; then decode + render timed
    def timed_fps(fn):
        gs = torch.cuda.Stream(device=dev)
        gs.wait_stream(stream)
        gg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gg, stream=gs):
            fn()
        stream.wait_stream(gs)
        for _ in range(Wm):
            gg.replay()
        barrier()
        for i in range(K):
            flush.zero_()
            s_ev[i].record(stream)
            gg.replay()
            e_ev[i].record(stream)
        barrier()
        return world * K / (max_over_ranks(sum(s_ev[i].elapsed_time(e_ev[i]) for i in range(K)))
                            / 1000.0)

    fpipe = Pipeline(N_GAUSS, W_IMG, H_IMG, 1, device=dev)
    fitted_state = {"render_fps": timed_fps(lambda: fpipe.render_frame(fitted))}
    fpipe.render_frame(fitted)
    torch.cuda.synchronize(dev)
    fitted_state["keys"] = fpipe.frame_keys()
    fp_host = fitted[0].cpu().numpy()
    lmin, lmax = fp_host[:, 2:5].min(axis=0), fp_host[:, 2:5].max(axis=0)
    c_gamma = [float(x) for x in np.maximum((lmax - lmin) / 63.0, 1e-6)]
    c_beta = [float(x) for x in lmin]
    cols = torch.from_numpy(np.ascontiguousarray(fp_host[:, 5:8])).to(dev)
    kws = torch.zeros(gi.gi_kmeans_workspace_bytes(8), dtype=torch.uint8, device=dev)
    asg = torch.zeros(N_GAUSS, dtype=torch.int32, device=dev)
    books = torch.zeros(2, 8, 3, dtype=torch.float32, device=dev)
    pts = cols
    for st in range(2):
        cent = pts[:: N_GAUSS // 8][:8].clone()
        for _ in range(5):
            gi.gi_kmeans_step(pts, cent, asg, kws)
        gi.gi_kmeans_step(pts, cent, asg, kws)        # final assignment for the residuals
        books[st] = cent
        pts = (pts - cent[asg.long()]).contiguous()   # stage-2 input: residuals
    cmeta = gi.codec_meta(N_GAUSS, c_gamma, c_beta, books)
    cpay = torch.zeros((N_GAUSS * 56 + 7) // 8 + 16, dtype=torch.uint8, device=dev)
    gi.gi_vq_encode(fitted[0].contiguous(), cmeta, cpay)
    cparams = torch.zeros(1, N_GAUSS, 8, dtype=torch.float32, device=dev)
    cpipe = Pipeline(N_GAUSS, W_IMG, H_IMG, 1, device=dev)
    fitted_state["decode_fps"] = timed_fps(lambda: cpipe.decode_render_frame(cpay, cmeta, cparams))
    dimg = cpipe.decode_render_frame(cpay, cmeta, cparams)
    fitted_state["psnr_db_fitted"] = float(fpipe.psnr(fpipe.render_frame(fitted), target)[0])
    fitted_state["psnr_db_decoded"] = float(cpipe.psnr(dimg, target)[0])
    fitted_state["bpp"] = 56.0 * N_GAUSS / (W_IMG * H_IMG)
    # the paper's remedy (Fig. 3): quantisation-aware fine-tuning,
    # then re-encode with the learned gamma / beta and EMA codebooks
    from paper_2403_08551_b200.pipeline import QatFitter
    qf = QatFitter(fitted[0].clone(), target, c_gamma, c_beta, books)
    for _ in range(2000):
        qf.step()
    torch.cuda.synchronize(dev)
    qp = qf.qparams.cpu().numpy()
    qmeta = gi.codec_meta(N_GAUSS, qp[:3], qp[3:], qf.books)
    gi.gi_vq_encode(qf.params, qmeta, cpay)
    dimg = cpipe.decode_render_frame(cpay, qmeta, cparams)
    fitted_state["psnr_db_decoded_after_qat2000"] = float(cpipe.psnr(dimg, target)[0])
    del psnr_pipe, fpipe, cpipe, qf

    # ---------------- fitting as a user runs it: 100 chained steps per graph, warm L2 ----
    # (context only: `value` above is the cold-L2 single-step number)
    wfit = Fitter(params.clone(), target)
    wfit.step()
    torch.cuda.synchronize(dev)
    wg = wfit.capture(100)
    wg.replay()
    barrier()
    s_ev[0].record(stream)
    for _ in range(3):
        wg.replay()
    e_ev[0].record(stream)
    barrier()
    warm_its = world * 300 / (max_over_ranks(s_ev[0].elapsed_time(e_ev[0])) / 1000.0)
    if wfit.check() != gi.GI_OK:
        raise RuntimeError("warm fit status")
    del wfit, wg

    # ---------------- NEXT-2: encoder (gi_vq_encode) and QAT step (gi_qat_step) ------------
    from paper_2403_08551_b200.pipeline import QatFitter
    fp = torch.from_numpy(synth.fitted_params(seed, N_GAUSS)).to(dev).contiguous()
    qgamma, qbeta = [0.05, 0.04, 0.05], [-1.0, -1.2, -1.0]
    qbooks = torch.from_numpy(np.random.default_rng(seed).normal(0, 0.3, (2, 8, 3))
                              .astype(np.float32)).to(dev)
    emeta = gi.codec_meta(N_GAUSS, qgamma, qbeta, qbooks)
    epay = torch.zeros((N_GAUSS * 56 + 7) // 8 + 16, dtype=torch.uint8, device=dev)
    eeff = torch.zeros(N_GAUSS, 8, dtype=torch.float32, device=dev)
    gi.gi_vq_encode(fp, emeta, epay, eeff)
    es = torch.cuda.Stream(device=dev)
    es.wait_stream(stream)
    eg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(eg, stream=es):
        gi.gi_vq_encode(fp, emeta, epay, eeff, stream=es)
    stream.wait_stream(es)
    for _ in range(Wm):
        eg.replay()
    barrier()
    for i in range(K):
        flush.zero_()
        s_ev[i].record(stream)
        eg.replay()
        e_ev[i].record(stream)
    barrier()
    enc_ms = max_over_ranks(sum(s_ev[i].elapsed_time(e_ev[i]) for i in range(K)))
    encode_fps = world * K / (enc_ms / 1000.0)
    qfit = QatFitter(fp.clone(), target, qgamma, qbeta, qbooks)
    qfit.step()
    torch.cuda.synchronize(dev)
    qg = qfit.capture(1)
    for _ in range(Wm):
        qg.replay()
    barrier()
    for i in range(K):
        flush.zero_()
        s_ev[i].record(stream)
        qg.replay()
        e_ev[i].record(stream)
    barrier()
    qat_ms = max_over_ranks(sum(s_ev[i].elapsed_time(e_ev[i]) for i in range(K)))
    qat_its = world * K / (qat_ms / 1000.0)
    if qfit.check() != gi.GI_OK:
        raise RuntimeError("qat status")
    del qfit, qg, eg

    # ---------------- batched launch (configs[3] pattern): B images per launch ------------
    batched = None
    B = args.batch_images if args.batch_images >= 0 else max(1, 64 // world)
    if B > 1:
        bp = torch.from_numpy(np.stack([synth.init_params(100 + B * rank + b, N_GAUSS)
                                        for b in range(B)])).to(dev).contiguous()
        bt = torch.from_numpy(np.stack([synth.image(100 + B * rank + b, W_IMG, H_IMG)
                                        for b in range(B)])).to(dev).contiguous()
        bfit = Fitter(bp.clone(), bt)
        bfit.step()
        torch.cuda.synchronize(dev)
        bplain = bfit.capture(1)
        bev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(6)]
        for e in bev:
            e.record(stream)
        torch.cuda.synchronize(dev)
        bstaged = bfit.capture(1, stage_events=bev)
        for _ in range(Wm):
            bplain.replay()
        KB = max(10, K // 4)
        barrier()
        for i in range(KB):
            flush.zero_()
            s_ev[i].record(stream)
            bplain.replay()
            e_ev[i].record(stream)
        barrier()
        b_ms = max_over_ranks(sum(s_ev[i].elapsed_time(e_ev[i]) for i in range(KB)))
        bk_ms = 0.0
        for i in range(min(KB, 20)):
            flush.zero_()
            bstaged.replay()
            torch.cuda.synchronize(dev)
            bk_ms += bev[2].elapsed_time(bev[3])
        bk_ms /= min(KB, 20)
        bpipe = Pipeline(N_GAUSS, W_IMG, H_IMG, B, device=dev)
        bpipe.project(bp)
        torch.cuda.synchronize(dev)
        bpairs = pairs_of(bpipe, np)
        brs = torch.cuda.Stream(device=dev)
        brs.wait_stream(stream)
        brg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(brg, stream=brs):
            bpipe.render_frame(bp)
        stream.wait_stream(brs)
        for _ in range(Wm):
            brg.replay()
        barrier()
        for i in range(KB):
            flush.zero_()
            s_ev[i].record(stream)
            brg.replay()
            e_ev[i].record(stream)
        barrier()
        br_ms = max_over_ranks(sum(s_ev[i].elapsed_time(e_ev[i]) for i in range(KB)))
        batched = {"workload": "configs[3]: 64 Kodak-shaped images (70k Gaussians each) sharded "
                               "over the ranks, each rank's share fit in one launch"
                               if args.batch_images < 0 else f"{B} C2 images per launch",
                   "images_per_launch": B, "images_total": world * B, "steps": KB,
                   "fit_image_its_per_s": world * B * KB / (b_ms / 1000.0),
                   "render_image_fps": world * B * KB / (br_ms / 1000.0),
                   "ms_per_fit_step": b_ms / KB, "fused_tile_kernel_ms": bk_ms,
                   "fused_tile_kernel_tflops": bpairs * FLOP_PER_PAIR_FUSED / (bk_ms * 1e-3) / 1e12,
                   "pixel_gaussian_pairs": bpairs}
        del bfit, bpipe, bplain, bstaged, brg

    # ---------------- e2e through the public API, host buffers ----------------
    # Every step copies its target image H2D from pinned host memory (on a copy
    # stream, double-buffered, so step i's copy overlaps step i-1's compute)
    # and reads its loss back D2H; L2 is still flushed before every step.
    # e2e = steps / device time of the whole pipelined run (events on the
    # compute stream; the copy stream is joined before the end event).
    pinned_t = torch.from_numpy(t_host).pin_memory()
    pinned_loss = torch.zeros(K + Wm, dtype=torch.float32).pin_memory()
    cstream = torch.cuda.Stream(device=dev)
    tbuf = [target.clone(), target.clone()]
    copied = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    e2e_fit = Fitter(params.clone(), tbuf[0])

    def e2e_run(nsteps, loss_off):
        cstream.wait_stream(stream)
        with torch.cuda.stream(cstream):
            tbuf[0].view(-1).copy_(pinned_t.view(-1), non_blocking=True)
            copied[0].record(cstream)
        for i in range(nsteps):
            b = i & 1
            if i + 1 < nsteps:
                with torch.cuda.stream(cstream):
                    if i >= 1:
                        cstream.wait_event(consumed[b ^ 1])
                    tbuf[b ^ 1].view(-1).copy_(pinned_t.view(-1), non_blocking=True)
                    copied[b ^ 1].record(cstream)
            flush.zero_()
            stream.wait_event(copied[b])
            e2e_fit.target = tbuf[b]
            # the loss read-back: the finalize kernel writes it straight into
            # pinned (UVA-mapped) host memory -- a copy-engine D2H per step
            # queues behind the next step's H2D and halves the rate
            e2e_fit.step(loss_out=pinned_loss[loss_off + i].data_ptr())
            consumed[b].record(stream)
        stream.wait_stream(cstream)

    e2e_run(Wm, 0)
    barrier()
    s_ev[0].record(stream)
    e2e_run(K, Wm)
    e_ev[0].record(stream)
    barrier()
    clk = clocks.stop()
    e2e_ms = s_ev[0].elapsed_time(e_ev[0])
    e2e_value = world * K / (max_over_ranks(e2e_ms) / 1000.0)
    e2e_losses = pinned_loss.numpy()[: K + Wm]
    if not (np.all(np.isfinite(e2e_losses)) and np.all(e2e_losses > 0)):
        raise RuntimeError("e2e losses missing or not finite")

    # ---------------- quality + the one collective (NCCL all-gather of PSNR) ----
    img = pipe.render_frame(fit.params)
    psnr = pipe.psnr(img, target).clone()
    # the one collective of the path: NCCL all-gather of per-image PSNR
    psnrs = gather_psnr(psnr, world, world, rank).tolist()

    if rank == 0:
        pk, pk_kind = peaks()
        sm_mhz = float(pk.get("sm_max_mhz", 1965.0))
        fp32_peak = 2 * FP32_LANES_PER_SM * N_SM * sm_mhz * 1e6 / 1e12     # TFLOP/s (FMA = 2)
        kern_ms = stage_ms[2]
        if batched is not None:
            batched["fused_tile_kernel_frac"] = batched["fused_tile_kernel_tflops"] / fp32_peak
        achieved = pairs * FLOP_PER_PAIR_FUSED / (kern_ms * 1e-3) / 1e12
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(prof):
            try:
                with open(prof) as f:
                    traffic = json.load(f).get("backward_tile_kernel_dram_bytes")
            except Exception:
                traffic = None
        ms_step = fit_ms_max / K
        line = {
            "metric": METRIC, "value": fit_value, "unit": "it/s", "n_gpus": world, "steps": K,
            "warmup": Wm, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": fit_value / world / PAPER_FIT_ITS if world == 1 else None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C2 (configs[1]): Kodak-shaped 768x512 synthetic image, 70k "
                                   "Gaussians at the paper's init, one Adam fit step "
                                   "(project+bin+fwd+L2+bwd+finalize+adam)",
                       "images_per_gpu": 1, "l2": "flushed (256 MB write) before every timed step",
                       "key_pairs_per_step": keys, "pixel_gaussian_pairs": pairs,
                       "vs_baseline_ref": "paper fit 469.1 it/s (Table 1a P:331, V100, Adan, "
                                          "real Kodak): context, other hardware"},
            "render_fps": render_fps,
            "fit_its_adan": adan_value,
            "fit_its_warm_graph100": warm_its,
            "fit_50k_steps": full_fit,
            "fitted_state": fitted_state,
            "fitted_note": "context: the cloud the 50k-step Adam fit produced -- render FPS, and "
                           "configs[4] decode + render of its C5 payload (fp16 positions, 6-bit "
                           "l codes, 2x8 RVQ colours by K-means, 56-bit records); PSNR before "
                           "and after the codec, without and with 2000 QAT steps (gi_qat_step)",
            "fit_50k_note": "the paper's training length (50k steps, P:381) on the C2 synthetic "
                            "image from the init cloud: device seconds per rank (max), PSNR of "
                            "the result; paper: 106.59 s on a V100 (Table 1a, P:331), context",
            "fit_warm_note": "context, not `value`: 100 chained Adam steps per CUDA graph "
                             "replay, no L2 flush between steps (a long fit as a user runs it)",
            "batched": batched,
            "decode_fps": decode_fps,
            "decode_fps_codec_sizes": decode_small,
            "encode_fps": encode_fps,
            "qat_its": qat_its,
            "next2_note": "encode_fps: gi_vq_encode of 70k fitted records (fp16 positions, "
                          "6-bit codes, 2x8 RVQ, packed 56-bit records + dequantised params); "
                          "qat_its: gi_qat_step on the C2 fitted proxy (quantise, fused fit "
                          "core, straight-through Adam, EMA codebooks)",
            "stage_ms": {"tile_kernel_fwd_l2_bwd": stage_ms[2],
                         "finalize_adam_next_projection_binning": stage_ms[3],
                         "event_overhead_empty_stages": stage_ms[0] + stage_ms[1],
                         "note": "chained step = 2 kernels; staged graph with event nodes "
                                 "(each costs a few us), so the stages add up to more than "
                                 "ms_per_step"},
            "render_kernel_ms": r_kernel_ms,
            "psnr_db_after_fit_steps": psnrs,
            "roofline": {"kernel": "backward_tile_kernel (fused Eq.7 fwd + L2 + App.A bwd)",
                         "bound": "alu", "achieved": achieved, "peak": fp32_peak,
                         "unit": "TFLOP/s", "frac": achieved / fp32_peak, "traffic": traffic,
                         "peak_kind": f"FP32 FMA pipe: 128 lanes x 2 FLOP x 148 SM x "
                                      f"{sm_mhz:.0f} MHz ({pk_kind} sm_max_mhz)",
                         "algorithmic": f"{FLOP_PER_PAIR_FUSED} FLOP per in-box pair x {pairs} "
                                        f"pairs per launch",
                         "render_kernel_frac": render_pairs * FLOP_PER_PAIR_RENDER
                         / (r_kernel_ms * 1e-3) / 1e12 / fp32_peak},
            "clocks": clk,
            "e2e": {"value": e2e_value, "unit": "it/s",
                    "h2d_bytes_per_step": int(t_host.nbytes), "d2h_bytes_per_step": 4,
                    "path": "Fitter.step -> gi_fit_step_chained (C ABI, no graph); per step: "
                            "H2D of the target from pinned host on a copy stream (double-"
                            "buffered, overlapping the previous step), L2 flush, fit step whose "
                            "finalize kernel writes the loss into pinned, UVA-mapped host "
                            "memory (the step's D2H); value = steps / device time; bound by "
                            "the host link (pinned H2D 22-37 GB/s across boxes)"},
            "gpu_launches": int(launches_per_step * K),
            "gpu_launches_per_step": int(launches_per_step),
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args.cpu_seconds)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def pairs_of(pipe, np_):
    rec = pipe.proj.view(-1, 12).cpu().numpy()
    bx, by = rec[:, 7].view(np_.uint32), rec[:, 11].view(np_.uint32)
    wx = (bx >> 16).astype(np_.int64) - (bx & 0xffff).astype(np_.int64) + 1
    wy = (by >> 16).astype(np_.int64) - (by & 0xffff).astype(np_.int64) + 1
    touched = pipe.tiles_touched.cpu().numpy() > 0
    return int(np_.sum(np_.where(touched, wx * wy, 0)))


if __name__ == "__main__":
    main()
