"""Device-resident buffers around the libgi C ABI: allocation (torch, once),
the render / fit-step sequences, and CUDA-graph capture of a fit step.

No arithmetic of the method lives here -- every step is a libgi call.
"""
from __future__ import annotations

import torch

from . import gi


def _u32(n: int, device) -> torch.Tensor:
    # uint32 storage; torch.int32 has the same bits and full op support
    return torch.zeros(max(int(n), 1), dtype=torch.int32, device=device)


def _bytes(n: int, device) -> torch.Tensor:
    # raw workspace of >= n bytes; torch allocations are >= 256-B aligned
    return torch.zeros(max((int(n) + 15) // 16, 1) * 4, dtype=torch.float32, device=device)


def default_capacity(n: int, batch: int) -> int:
    """Generous key capacity: 16 tiles per Gaussian on average (the paper's
    init touches ~1.8, a 3x-larger fitted cloud ~4.5), at least 64 Ki."""
    return max(1 << 16, 16 * int(n) * int(batch))


class Pipeline:
    """All buffers of one (n, W, H, batch) problem on one device."""

    def __init__(self, n: int, width: int, height: int, batch: int = 1, k: float = 3.0,
                 key_capacity: int | None = None, device: str | torch.device = "cuda"):
        gi.load()
        self.device = torch.device(device)
        self.n, self.W, self.H, self.B = int(n), int(width), int(height), int(batch)
        self.f = gi.frame(width, height, batch, k)
        self.T = gi.gi_num_tiles(self.f)
        self.cap = int(key_capacity) if key_capacity else default_capacity(n, batch)
        d = self.device
        tot = self.n * self.B
        self.proj = torch.zeros(max(tot, 1) * gi.GI_PROJ_BYTES // 4, dtype=torch.float32, device=d)
        self.tiles_touched = _u32(tot, d)
        self.key_tile = _u32(self.cap, d)
        self.key_gid = _u32(self.cap, d)
        self.tile_range = _u32(self.T * self.B + 1, d)
        self.n_keys = _u32(1, d)
        self.bin_ws = _bytes(gi.gi_bin_workspace_bytes(n, self.cap, self.f), d)
        self.bwd_ws = _bytes(gi.gi_backward_workspace_bytes(n, self.cap, self.f), d)
        self.psnr_ws = _bytes(gi.gi_psnr_workspace_bytes(self.f), d)
        self.image = torch.zeros(self.B, 3, self.H, self.W, dtype=torch.float32, device=d)
        self.grads = torch.zeros(self.B, max(self.n, 1), 8, dtype=torch.float32, device=d)
        self.loss = torch.zeros(self.B, dtype=torch.float32, device=d)
        self.psnr_out = torch.zeros(self.B, dtype=torch.float32, device=d)
        self.flags_word = _u32(1, d)

    # -- stages -----------------------------------------------------------
    def project(self, params, flags=gi.GI_POS_LOGIT, stream=None):
        gi.gi_project(params, self.n, self.f, flags, self.proj, self.tiles_touched, stream)

    def bin(self, stream=None):
        gi.gi_bin(self.proj, self.tiles_touched, self.n, self.f, self.cap, self.bin_ws,
                  self.key_tile, self.key_gid, self.tile_range, self.n_keys, stream)

    def raster(self, stream=None):
        gi.gi_render(self.proj, self.key_gid, self.tile_range, self.n, self.f, self.image, stream)

    def render(self, params, flags=gi.GI_POS_LOGIT, stream=None) -> torch.Tensor:
        """project -> bin -> render (Eq. 7); returns the [B][3][H][W] image buffer."""
        self.project(params, flags, stream)
        self.bin(stream)
        self.raster(stream)
        return self.image

    def render_frame(self, params, flags=gi.GI_POS_LOGIT, stream=None) -> torch.Tensor:
        """Fused gi_render_frame (project + counts -> bin -> render with the
        per-tile ordering inside the render kernel) into self.image."""
        if not hasattr(self, "frame_ws"):
            self.frame_ws = _bytes(gi.gi_fit_workspace_bytes(self.n, self.cap, self.f), self.device)
        gi.gi_render_frame(params, self.n, self.f, flags, self.cap, self.frame_ws, self.image, stream)
        return self.image

    def decode_render_frame(self, payload, meta, params_out=None, stream=None) -> torch.Tensor:
        """configs[4]: gi_decode_render_frame (decode fused into the
        projection, then render) into self.image; params_out optional."""
        if not hasattr(self, "frame_ws"):
            self.frame_ws = _bytes(gi.gi_fit_workspace_bytes(self.n, self.cap, self.f), self.device)
        gi.gi_decode_render_frame(payload, meta, self.f, self.cap, self.frame_ws, self.image,
                                  params_out, stream)
        return self.image

    def frame_keys(self) -> int:
        ptr = gi.gi_fit_n_keys(self.frame_ws, self.n, self.cap, self.f)
        off = (ptr - self.frame_ws.data_ptr()) // 4
        return int(self.frame_ws.view(torch.int32)[off].item()) & 0xffffffff

    def backward(self, params, target=None, dL_dimage=None, flags=gi.GI_POS_LOGIT,
                 image_out=None, stream=None) -> torch.Tensor:
        """Fused forward + L2 + backward on the current bins (after project/bin)."""
        gi.gi_render_backward(params, self.proj, self.key_gid, self.tile_range,
                              self.n, self.f, flags, dL_dimage, target, self.cap, self.bwd_ws,
                              self.grads, self.loss if dL_dimage is None else None, image_out,
                              stream)
        return self.grads

    def psnr(self, image, target, stream=None) -> torch.Tensor:
        gi.gi_psnr(image, target, self.f, self.psnr_out, self.psnr_ws, stream)
        return self.psnr_out

    def check(self, stream=None) -> int:
        return gi.gi_check(self.n_keys, self.cap, self.flags_word, stream)

    def keys(self) -> int:
        return int(self.n_keys[0].item()) & 0xffffffff


class Fitter:
    """Adam fitting loop over B images with the device-resident fused step
    (gi_fit_step), optionally replayed from a captured CUDA graph."""

    def __init__(self, params: torch.Tensor, target: torch.Tensor, k: float = 3.0,
                 key_capacity: int | None = None, lr0: float = 1e-3, half_every: int = 20000,
                 beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                 flags: int = gi.GI_POS_LOGIT, chained: bool = True, optimizer: str = "adam",
                 beta3: float = 0.99, weight_decay: float = 0.0):
        """optimizer: "adam" (north_star) or "adan" (the paper's, P:381;
        default betas (0.98, 0.92, 0.99) when beta1/beta2 are left at Adam's
        defaults); either is fused into the finalize kernel, chained or not."""
        gi.load()
        if optimizer not in ("adam", "adan"):
            raise ValueError("optimizer must be 'adam' or 'adan'")
        self.optimizer = optimizer
        if optimizer == "adan" and (beta1, beta2) == (0.9, 0.999):
            beta1, beta2 = 0.98, 0.92
        self.chained = bool(chained)
        self.primed = False
        assert params.dim() == 3 and params.shape[2] == 8, "params [B][N][8]"
        B, n = params.shape[0], params.shape[1]
        H, W = target.shape[-2], target.shape[-1]
        self.device = params.device
        self.params = params.contiguous()
        self.target = target.contiguous()
        self.n, self.B = n, B
        self.f = gi.frame(W, H, B, k)
        self.cap = int(key_capacity) if key_capacity else default_capacity(n, B)
        self.fit_ws = _bytes(gi.gi_fit_workspace_bytes(n, self.cap, self.f), self.device)
        self.grads = torch.zeros_like(self.params)
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.step_counter = _u32(1, self.device)
        self.status = _u32(1, self.device)
        self.loss = torch.zeros(B, dtype=torch.float32, device=self.device)
        self.hyper = dict(lr0=lr0, half_every=half_every, beta1=beta1, beta2=beta2, eps=eps)
        if optimizer == "adan":
            self.n_acc = torch.zeros_like(self.params)
            self.grad_prev = torch.zeros_like(self.params)
            self.adan_extra = dict(beta3=beta3, weight_decay=weight_decay)
        self.flags = flags
        self.graph = None
        self._call = None                       # prepared gi.FitStepCall (Adam, built on first step)
        self._call_key = None
        self._tshape = self.target.shape

    def step(self, stream=None, stage_events=None, loss_out=None):
        """One fused step.  In chained mode (default) the first call primes
        the workspace and every step fuses the next step's projection into
        its Adam kernel; the params must not be written by anyone else in
        between (call unchain() after modifying them).  loss_out: where the
        per-image losses go instead of self.loss -- e.g. the address of
        pinned host memory, which the finalize kernel then writes directly
        (mapped, no copy-engine transfer)."""
        loss = self.loss if loss_out is None else loss_out
        if self.chained and not self.primed:
            gi.gi_fit_prime(self.params, self.n, self.f, self.flags, self.cap, self.fit_ws, stream)
            self.primed = True
        if self.optimizer == "adan":
            fn = gi.gi_fit_step_adan_chained if self.chained else gi.gi_fit_step_adan
            fn(self.params, self.grads, self.m, self.v, self.n_acc, self.grad_prev, self.target,
               self.n, self.f, self.flags, self.cap, self.fit_ws, self.step_counter, loss=loss,
               status_flags=self.status, stream=stream, **self.hyper, **self.adan_extra)
            return
        if stage_events is None:
            # the prepared call (gi.FitStepCall): same entry point, arguments
            # marshalled once per Fitter
            key = (self.params.data_ptr(), self.grads.data_ptr(), self.m.data_ptr(),
                   self.v.data_ptr(), self.fit_ws.data_ptr())
            if self._call is None or self._call_key != key:    # (re)built if a buffer was replaced
                self._call_key = key
                h = self.hyper
                self._call = gi.FitStepCall(self.chained, self.params, self.grads, self.m, self.v,
                                            self.n, self.f, self.flags, self.cap, self.fit_ws,
                                            self.step_counter, h["lr0"], h["half_every"],
                                            h["beta1"], h["beta2"], h["eps"], self.status)
            t = self.target
            if not (t.is_cuda and t.is_contiguous() and t.shape == self._tshape):
                raise ValueError("target: a contiguous device tensor [B][3][H][W]")
            self._call(t.data_ptr(), loss if isinstance(loss, int) else gi._ptr(loss),
                       gi._stream(stream))
        elif self.chained:
            gi.gi_fit_step_chained(self.params, self.grads, self.m, self.v, self.target, self.n,
                                   self.f, self.flags, self.cap, self.fit_ws, self.step_counter,
                                   loss=loss, status_flags=self.status,
                                   stage_events=stage_events, stream=stream, **self.hyper)
        else:
            gi.gi_fit_step(self.params, self.grads, self.m, self.v, self.target, self.n, self.f,
                           self.flags, self.cap, self.fit_ws, self.step_counter, loss=loss,
                           status_flags=self.status, stage_events=stage_events, stream=stream,
                           **self.hyper)

    def unchain(self):
        """Params were modified externally: re-prime before the next chained step."""
        self.primed = False

    def capture(self, steps_per_graph: int = 1, stage_events=None):
        """Capture `steps_per_graph` fused steps into one CUDA graph (stage
        events, if given, are recorded around the last captured step).  In
        chained mode the workspace is primed (eagerly) first."""
        if self.chained and not self.primed:
            gi.gi_fit_prime(self.params, self.n, self.f, self.flags, self.cap, self.fit_ws)
            self.primed = True
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(steps_per_graph):
                self.step(stage_events=stage_events if i == steps_per_graph - 1 else None)
        torch.cuda.current_stream(self.device).wait_stream(s)
        self.graph = g
        self.steps_per_graph = steps_per_graph
        self._graphs = getattr(self, "_graphs", []) + [g]   # keep every captured graph alive
        return g

    def replay(self):
        self.graph.replay()

    def n_keys(self) -> int:
        ptr = gi.gi_fit_n_keys(self.fit_ws, self.n, self.cap, self.f)
        base = self.fit_ws.data_ptr()
        off = (ptr - base) // 4
        return int(self.fit_ws.view(torch.int32)[off].item()) & 0xffffffff

    def seg_stats(self) -> tuple[int, int]:
        """(tiles streamed past their slab, tiles past the sort buffer) since
        the last prime / reset / non-chained step."""
        ptr = gi.gi_fit_seg_stats(self.fit_ws, self.n, self.cap, self.f)
        off = (ptr - self.fit_ws.data_ptr()) // 4
        w = self.fit_ws.view(torch.int32)[off:off + 2].cpu().tolist()
        return int(w[0]) & 0xffffffff, int(w[1]) & 0xffffffff

    def check(self) -> int:
        # direct binning has no hard key capacity (overflowing tiles are
        # streamed), so only the device status word is checked
        return gi.gi_check(None, self.cap, self.status)

    def steps_done(self) -> int:
        return int(self.step_counter[0].item())

    # -- checkpoint / resume ---------------------------------------------------
    _STATE = ("params", "m", "v", "n_acc", "grad_prev")

    def save(self, path: str) -> None:
        """Checkpoint: params and the optimiser state (Adam m, v;
        Adan also n and the previous gradient), the device step counter and
        the hyper-parameters, as one .npz of the raw fp32 / u32 bits.  Resuming
        from it continues the fit bit for bit (`Fitter.load`)."""
        import numpy as np
        torch.cuda.synchronize(self.device)
        arrays = {k: getattr(self, k).cpu().numpy() for k in self._STATE if hasattr(self, k)}
        arrays["step_counter"] = self.step_counter.cpu().numpy()
        meta = dict(optimizer=self.optimizer, flags=int(self.flags), k=float(self.f.k),
                    width=int(self.f.width), height=int(self.f.height), batch=int(self.B),
                    n=int(self.n), key_capacity=int(self.cap), chained=bool(self.chained),
                    **{k: float(v) for k, v in self.hyper.items()},
                    **({k: float(v) for k, v in self.adan_extra.items()}
                       if self.optimizer == "adan" else {}))
        arrays["meta_json"] = np.frombuffer(__import__("json").dumps(meta).encode(), np.uint8)
        np.savez(path, **arrays)

    @classmethod
    def load(cls, path: str, target: torch.Tensor) -> "Fitter":
        """A Fitter resumed from `save(path)` on `target`'s device (the target
        image is not part of the checkpoint).  The next step re-primes (chained
        mode) from the restored params, so the trajectory equals the one the
        saving Fitter would have followed."""
        import json

        import numpy as np
        z = np.load(path)
        meta = json.loads(bytes(z["meta_json"]).decode())
        dev = target.device
        params = torch.from_numpy(z["params"]).to(dev)
        kw = dict(k=meta["k"], key_capacity=meta["key_capacity"], lr0=meta["lr0"],
                  half_every=int(meta["half_every"]), beta1=meta["beta1"], beta2=meta["beta2"],
                  eps=meta["eps"], flags=meta["flags"], chained=meta["chained"],
                  optimizer=meta["optimizer"])
        if meta["optimizer"] == "adan":
            kw.update(beta3=meta["beta3"], weight_decay=meta["weight_decay"])
        f = cls(params, target, **kw)
        if (f.f.width, f.f.height, f.B, f.n) != (meta["width"], meta["height"], meta["batch"],
                                                   meta["n"]):
            raise ValueError("checkpoint does not match the target's frame")
        for k in cls._STATE:
            if k in z.files and k != "params":
                getattr(f, k).copy_(torch.from_numpy(z[k]).to(dev))
        f.step_counter.copy_(torch.from_numpy(z["step_counter"]).to(dev))
        return f

    # -- a logged fit loop -------------------------------------------------------
    def fit(self, steps: int, log_every: int = 100, log=None, psnr: bool = True) -> list:
        """Run `steps` fused steps, `log_every` per CUDA-graph replay, and at
        every log point check the device status (GI_ENONFINITE raises) and
        record {"step", "loss", "psnr_db", "it_per_s"} -- one JSON object per
        line to `log` (a path or a writable text file) if given (SURVEY §5:
        PSNR, loss and it/s as JSONL; SPEC logs every 100 steps).  Returns the
        records."""
        import json
        import time
        rec, fh, own = [], None, False
        if isinstance(log, str):
            fh, own = open(log, "a"), True
        elif log is not None:
            fh = log
        pipe = Pipeline(self.n, self.f.width, self.f.height, self.B, self.f.k, self.cap,
                        self.device) if psnr else None
        full, rem = divmod(int(steps), int(log_every))
        g = self.capture(log_every) if full else None
        try:
            t0 = time.perf_counter()
            for chunk in [log_every] * full + ([rem] if rem else []):
                if chunk == log_every:
                    g.replay()
                else:
                    for _ in range(chunk):
                        self.step()
                st = self.check()
                if st != gi.GI_OK:
                    raise gi.GiError(st, "Fitter.fit", "non-finite parameters or gradients")
                t1 = time.perf_counter()
                r = {"step": self.steps_done(), "loss": [float(x) for x in self.loss.cpu()],
                     "it_per_s": chunk / max(t1 - t0, 1e-9)}
                if pipe is not None:
                    img = pipe.render_frame(self.params, self.flags)
                    r["psnr_db"] = [float(x) for x in pipe.psnr(img, self.target).cpu()]
                rec.append(r)
                if fh is not None:
                    fh.write(json.dumps(r) + "\n")
                    fh.flush()
                t0 = time.perf_counter()
        finally:
            if own:
                fh.close()
        return rec


class QatFitter:
    """NEXT-2 attribute quantisation-aware fine-tuning (gi_qat_step) of one
    image's fitted cloud: fp16 positions, b-bit Cholesky codes with learned
    gamma/beta, M-stage RVQ colours with EMA codebooks."""

    def __init__(self, params: torch.Tensor, target: torch.Tensor, gamma, beta,
                 books: torch.Tensor, k: float = 3.0, key_capacity: int | None = None,
                 **cfg):
        gi.load()
        assert params.dim() == 2 and params.shape[1] == 8, "params [N][8] (one image)"
        self.device = params.device
        n = params.shape[0]
        H, W = target.shape[-2], target.shape[-1]
        self.n = n
        self.f = gi.frame(W, H, 1, k)
        self.cfg = gi.qat_config(**cfg)
        self.cap = int(key_capacity) if key_capacity else default_capacity(n, 1)
        self.ws = _bytes(gi.gi_qat_workspace_bytes(n, self.cap, self.f, self.cfg), self.device)
        self.params = params.contiguous()
        self.target = target.contiguous()
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.eff = torch.zeros_like(self.params)
        self.grads = torch.zeros_like(self.params)
        self.qparams = torch.tensor(list(gamma) + list(beta), dtype=torch.float32,
                                    device=self.device)
        self.qm = torch.zeros(6, dtype=torch.float32, device=self.device)
        self.qv = torch.zeros(6, dtype=torch.float32, device=self.device)
        self.books = books.contiguous().clone()
        M, Bk = self.books.shape[0], self.books.shape[1]
        self.ema_n = torch.ones(M, Bk, dtype=torch.float32, device=self.device)
        self.ema_s = self.books.clone()
        self.step_counter = _u32(1, self.device)
        self.status = _u32(1, self.device)
        self.losses = torch.zeros(9, dtype=torch.float32, device=self.device)
        self.graph = None

    def step(self, stream=None):
        gi.gi_qat_step(self.params, self.m, self.v, self.eff, self.grads, self.qparams, self.qm,
                       self.qv, self.books, self.ema_n, self.ema_s, self.target, self.n, self.f,
                       self.cfg, self.cap, self.ws, self.step_counter, self.losses, self.status,
                       stream)

    def capture(self, steps_per_graph: int = 1):
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(steps_per_graph):
                self.step(s)
        torch.cuda.current_stream(self.device).wait_stream(s)
        self.graph = g
        return g

    def replay(self):
        self.graph.replay()

    def check(self) -> int:
        return gi.gi_check(None, self.cap, self.status)

