"""Worked examples of the paper / SPEC, stored as cited text fixtures under
tests/golden/, checked against the oracle (``-m "not gpu"``) and, where the
CUDA path computes the same quantity, against libgi (``-m gpu``)."""
import json
import math
import os

import numpy as np
import pytest

import synth

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(G, name)) as f:
        d = json.load(f)
    assert d["cite"] and d["cases"]
    return d["cases"]


def sym3(m):
    return [m[0][0], m[0][1], m[1][1]]


def centred(W, H, px, py, dx, dy, raw_l, colour):
    """One Gaussian, normalised position, centre at pixel (px, py)'s centre
    minus (dx, dy) (R1: pixel centres at +1/2)."""
    mx, my = px + 0.5 - dx, py + 0.5 - dy
    return np.array([[2 * mx / W - 1, 2 * my / H - 1, *raw_l, *colour]], np.float32)


# ------------------------------------------------------------------ oracle
def test_golden_covariance_inverse_sigma(gio):
    for c in load("covariance.json"):
        mode = 1 | (2 if c["kind"] == "rs" else 0)
        p = np.array([[0, 0, *c["raw"], 1, 1, 1]], np.float32)
        got = gio.project(p, 64, 64, pos_mode=mode)["sigma"][0]
        assert np.allclose(got, sym3(c["sigma"]), atol=1e-12), c
    for c in load("inverse.json"):
        assert np.allclose(gio.inverse2(sym3(c["sigma"])), sym3(c["inverse"]), atol=1e-15)
    for c in load("sigma.json"):
        assert gio.eval_sigma(sym3(c["sinv"]), *c["d"]) == c["sigma"]


def test_golden_position(gio):
    for c in load("position.json"):
        p = np.array([[*c["raw"], 0.5, 0, 0.5, 1, 1, 1]], np.float32)
        mu = gio.project(p, c["W"], c["H"])["mu"][0]
        assert np.allclose(mu, c["pixel"], atol=1e-4), (mu, c)   # fp32 raw atanh


def test_golden_render_and_backward_pixel(gio):
    for c in load("render.json"):
        px, py = c["centre_pixel"]
        p = centred(c["W"], c["H"], px, py, 0, 0, c["raw_l"], c["colour"])
        img = gio.render(p, c["W"], c["H"], pos_mode=gio.POS_NORMALIZED, mode=gio.DENSE)
        assert np.allclose(img[:, py, px], c["colour"], atol=1e-6)
    for c in load("backward_pixel.json"):
        # Sigma = I (raw l = (0.5, 0, 0.5)), d = pixel - mu = (1, 0), upstream at one pixel
        W, H, px, py = 8, 8, 4, 4
        p = centred(W, H, px, py, *c["d"], [0.5, 0.0, 0.5], c["colour"])
        up = np.zeros((3, H, W))
        up[:, py, px] = c["upstream"]
        g = gio.backward(p, up, W, H, pos_mode=gio.POS_NORMALIZED, mode=gio.DENSE)[0]
        assert np.allclose(g[5:8], c["dcolour"], atol=1e-6)
        # dC/dmu = -c' e^-sigma dsigma/dmu = c' e^-sigma Sigma^-1 d (R13);
        # with upstream (1, 0, 0): d/du_x = W/2 * e^-0.5 * d_x
        assert abs(g[0] - W / 2 * -c["dsigma"] * c["d"][0]) <= 1e-6
        assert abs(g[1]) <= 1e-9


def test_golden_chain_rules(gio):
    for c in load("chol_backward.json"):
        assert list(gio.chol_backward(sym3(c["G"]), *c["l_eff"])) == c["dl"]
    for c in load("rs_backward.json"):
        d = gio.rs_backward(sym3(c["G"]), c["theta"], *c["s_eff"])
        assert abs(d[0] - c["dtheta"]) <= 1e-12
        if "ds" in c:
            assert np.allclose(d[1:], c["ds"], atol=1e-12)


def test_golden_loss_lr_psnr(gio):
    for c in load("loss.json"):
        loss, g = gio.mse(np.array([[[c["rendered"]]]] * 3), np.full((3, 1, 1), c["target"],
                                                                   np.float32))
        assert loss == c["loss"] and np.allclose(g, c["upstream"] / 3.0)   # mean over 3HW
    for c in load("lr.json"):
        assert gio.lr_at(c["step"]) == c["lr"]
    for c in load("psnr.json"):
        x = np.full((3, 4, 4), 0.5)
        y = (x + math.sqrt(c["mse"])).astype(np.float32)
        assert abs(gio.psnr(x, y) - c["psnr"]) <= 1e-5


def test_golden_codec(gio):
    for c in load("quant.json"):
        p = np.array([[0, 0, c["l"], c["l"], c["l"], 0, 0, 0]], np.float32)
        e = gio.vq_encode(p, [c["gamma"]] * 3, [c["beta"]] * 3, np.zeros((2, 8, 3), np.float32),
                          bits=c["bits"], pos_mode=1)
        assert e["codes"].tolist() == [[c["code"]] * 3]
        assert np.allclose(e["eff"][0, 2:5], c["dequant"], atol=1e-6)
    for c in load("rvq.json"):
        p = np.array([[0, 0, 0, 0, 0, *c["colour"]]], np.float32)
        e = gio.vq_encode(p, [1] * 3, [0] * 3, np.float32(c["books"]), stages=c["M"],
                          codebook=c["B"], pos_mode=1)
        assert e["idx"].tolist() == [c["idx"]] and np.allclose(e["eff"][0, 5:], c["chat"])
    for c in load("record.json"):
        bits = c["bits_string"]
        assert len(bits) == c["record_bits"] == synth.record_bits(6, 2, 8)
        data = np.frombuffer(int(bits, 2).to_bytes(len(bits) // 8, "big"), np.uint8)
        books = np.zeros((2, 8, 3), np.float32)
        for m, k, v in c["book_entries"]:
            books[m, k] = v
        out = gio.vq_decode(data, 1, np.float32(c["gamma"]), np.float32(c["beta"]), books)[0]
        assert np.allclose(out, c["params"], atol=1e-6)


# --------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_golden_on_gpu(gi):
    import torch

    from paper_2403_08551_b200.pipeline import Pipeline
    dev = "cuda"
    for c in load("render.json"):
        px, py = c["centre_pixel"]
        p = centred(c["W"], c["H"], px, py, 0, 0, c["raw_l"], c["colour"])
        pipe = Pipeline(1, c["W"], c["H"], 1, device=dev)
        img = pipe.render(torch.from_numpy(p).to(dev)[None].contiguous(), gi.GI_POS_NORMALIZED)
        torch.cuda.synchronize()
        assert np.allclose(img[0, :, py, px].cpu().numpy(), c["colour"], atol=2e-6)
    for c in load("lr.json"):
        assert gi.gi_lr_at(c["step"]) == c["lr"]
    for c in load("record.json"):
        bits = c["bits_string"]
        data = torch.from_numpy(np.frombuffer(int(bits, 2).to_bytes(len(bits) // 8, "big"),
                                              np.uint8).copy()).to(dev)
        books = np.zeros((2, 8, 3), np.float32)
        for m, k, v in c["book_entries"]:
            books[m, k] = v
        bk = torch.from_numpy(books).to(dev)
        meta = gi.codec_meta(1, c["gamma"], c["beta"], bk)
        out = torch.zeros(1, 8, device=dev)
        gi.gi_vq_decode(data, meta, out)
        assert np.allclose(out[0].cpu().numpy(), c["params"], atol=1e-6)
        # and the encoder reproduces the record bit for bit
        pay = torch.zeros(8, dtype=torch.uint8, device=dev)
        gi.gi_vq_encode(out, meta, pay, None, flags=gi.GI_POS_NORMALIZED)
        torch.cuda.synchronize()
        assert bytes(pay[:7].cpu().numpy()) == bytes(data.cpu().numpy())
    for c in load("quant.json"):
        p = torch.tensor([[0, 0, c["l"], c["l"], c["l"], 0, 0, 0]], dtype=torch.float32, device=dev)
        bk = torch.zeros(2, 8, 3, device=dev)
        meta = gi.codec_meta(1, [c["gamma"]] * 3, [c["beta"]] * 3, bk, bits=c["bits"])
        eff = torch.zeros(1, 8, device=dev)
        gi.gi_vq_encode(p, meta, None, eff, flags=gi.GI_POS_NORMALIZED)
        torch.cuda.synchronize()
        assert np.allclose(eff[0, 2:5].cpu().numpy(), c["dequant"], atol=1e-6)
