"""Pins the oracle's DECLARED ALIF and RLIF cells (CPU only).

ALIF and RLIF are not in the reference,
so there is no
reference output to pin it to.  The oracle's restatement
(oracle/spiketrain_oracle.h, `cell`) is pinned instead against an independent
derivation: torch autograd (float64) of the same declared forward equations,
with the surrogate as a custom backward.  The oracle's hand-written reverse
scan must reproduce autograd's gradient for every entry, including the new
`l{id}.gamma` entries, the clip masks and the scalar BetaMode broadcast.
"""
import math

import numpy as np
import pytest
import torch

from oracle.pyoracle import Net


def _surrogate(act, k, aux, x):
    if act == "superspike":
        return 1.0 / (1.0 + k * x.abs()) ** 2
    if act == "arctan":
        u = math.pi * k * x / 2.0
        return 1.0 / (1.0 + u * u)
    if act == "triangular":
        return torch.clamp(1.0 - (k * x).abs(), min=0.0)
    if act == "boxcar":
        return torch.where(x.abs() <= k / 2.0, torch.full_like(x, aux), torch.zeros_like(x))
    return torch.ones_like(x)


class _Spike(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, act, k, aux):
        ctx.save_for_backward(x)
        ctx.cfg = (act, k, aux)
        return (x >= 0).to(x.dtype)

    @staticmethod
    def backward(ctx, g):
        (x,) = ctx.saved_tensors
        return g * _surrogate(*ctx.cfg, x), None, None, None


def _autograd(net: Net, entries, params, x, y, k, aux):
    """Loss and gradient of the declared network in float64 autograd."""
    P = {n: torch.tensor(params[o:o + s].astype(np.float64), requires_grad=True)
         for n, o, s in entries}
    names = [n for n, _, _ in entries]
    ws = [n for n in names if n.endswith(".w")]
    B, T, _ = x.shape
    a_in = torch.tensor(x.astype(np.float64))
    rasters = []
    for l, h in enumerate(net.hidden):
        lin = ws[l][:-2]
        cell = names[names.index(ws[l]) + (2 if net.bias else 1)][:-5]
        W = P[ws[l]].reshape(-1, h)
        cur = a_in @ W
        if net.bias:
            cur = cur + P[lin + ".b"]
        beta = P[cell + ".beta"]
        bc = torch.clamp(beta, 0.0, 1.0).expand(h) if beta.numel() == 1 else torch.clamp(beta, 0.0, 1.0)
        kind = (net.cell + ("lif",) * 8)[l]
        alif = kind == "alif"
        gc = torch.clamp(P[cell + ".gamma"], 0.0, 1.0) if alif else None
        rec = P[cell + ".rec"].reshape(h, h) if kind == "rlif" else None
        v = torch.zeros(B, h, dtype=torch.float64)
        a = torch.zeros(B, h, dtype=torch.float64)
        out = []
        for t in range(T):
            th = net.threshold + a if alif else torch.full_like(v, net.threshold)
            s = _Spike.apply(v - th, net.act, k, aux)
            v = v * bc + cur[:, t] - s * th
            if rec is not None:
                v = v + s @ rec
            if alif:
                a = a * gc + (1.0 - gc) * s
            out.append(s)
        a_in = torch.stack(out, 1)
        rasters.append(a_in.detach().numpy())
    W = P[ws[-1]].reshape(-1, net.classes)
    cur = a_in @ W
    if net.bias:
        cur = cur + P[ws[-1][:-2] + ".b"]
    beta = P[names[-1]]
    bc = torch.clamp(beta, 0.0, 1.0)
    v = torch.zeros(B, net.classes, dtype=torch.float64)
    logits = torch.zeros(B, net.classes, dtype=torch.float64)
    for t in range(T):
        v = v * bc + cur[:, t]
        logits = logits + v
    loss = torch.nn.functional.cross_entropy(logits, torch.tensor(y))
    loss.backward()
    g = np.zeros(params.size, np.float64)
    for n, o, s in entries:
        g[o:o + s] = P[n].grad.numpy() if P[n].grad is not None else 0.0
    return float(loss.detach()), g, rasters


CASES = [
    dict(hidden=(24, 16), cell=("alif", "alif"), act="superspike"),
    dict(hidden=(24, 16), cell=("alif", "lif"), act="arctan", bias=True),
    dict(hidden=(20,), cell=("alif",), act="triangular", beta_mode=("scalar", "per_neuron")),
    dict(hidden=(16, 16, 12), cell=("lif", "alif", "alif"), act="boxcar", threshold=0.8),
    dict(hidden=(24, 16), cell=("rlif", "rlif"), act="superspike"),
    dict(hidden=(20, 18), cell=("rlif", "lif"), act="arctan", bias=True, beta_mode=("scalar",)),
    dict(hidden=(16, 16, 12), cell=("alif", "rlif", "lif"), act="triangular"),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_alif_oracle_matches_autograd(orc, case):
    kw = dict(CASES[case])
    net = Net(inp=40, classes=5, unroll=7, **kw)
    B, T = 6, 30
    rng = np.random.default_rng(case)
    x = (rng.random((B, T, net.inp)) < 0.25).astype(np.uint8)
    y = rng.integers(0, net.classes, B).astype(np.int64)
    entries = orc.entries(net)
    assert any(n.endswith((".gamma", ".rec")) for n, _, _ in entries)
    params = orc.init(net, orc.key_child(orc.key_from_seed(case), 0))
    # louder weights so every layer spikes (and adapts) at a healthy rate
    for n, o, s in entries:
        if n.endswith(".w"):
            params[o:o + s] *= 3.0
    pk = orc.pack_time(x)
    ref = orc.forward_backward(net, params, pk, T, y, want_spikes=True)
    k, aux = net.c().slope, net.c().aux
    loss, g, rasters = _autograd(net, entries, params, x, y, k, aux)
    for l, r in enumerate(rasters):
        assert np.array_equal(ref["spikes"][l].astype(np.float64), r), f"raster {l} differs"
        assert 0.02 < r.mean() < 0.9, r.mean()
    assert abs(ref["loss"] - loss) <= 1e-5 * abs(loss)
    for n, o, s in entries:
        gr, go = g[o:o + s], ref["grads"][o:o + s].astype(np.float64)
        den = max(np.linalg.norm(gr), 1e-8)
        assert np.linalg.norm(go - gr) / den <= 2e-5, (n, np.linalg.norm(go - gr) / den)
    gam = [o for n, o, s in entries if n.endswith((".gamma", ".rec"))]
    assert any(np.abs(ref["grads"][o:o + 4]).max() > 0 for o in gam)


def test_alif_entries_and_init(orc):
    net = Net(inp=10, hidden=(8, 6), classes=3, cell=("alif", "lif"), monitor=(0,))
    e = orc.entries(net)
    assert [n for n, _, _ in e] == ["l0.w", "l1.beta", "l1.gamma", "l3.w", "l4.beta",
                                   "l5.w", "l6.beta"]
    p = orc.init(net, 1234)
    cell_key = orc.key_child(1234, 1)
    _, o, s = e[2]
    assert np.array_equal(p[o:o + s], orc.truncated_normal(orc.key_child(cell_key, 3), 8, 0.5, 0.25))
    _, o, s = e[1]
    assert np.array_equal(p[o:o + s], orc.truncated_normal(orc.key_child(cell_key, 2), 8, 0.5, 0.25))


def test_alif_without_adaptation_is_lif(orc):
    """gamma = 1 (clip) keeps a = 0: ALIF then reduces to the reference LIF bit for bit."""
    lif = Net(inp=30, hidden=(16,), classes=4)
    alif = Net(inp=30, hidden=(16,), classes=4, cell=("alif",))
    B, T = 5, 25
    rng = np.random.default_rng(7)
    pk = orc.pack_time((rng.random((B, T, 30)) < 0.3).astype(np.uint8))
    y = rng.integers(0, 4, B).astype(np.int64)
    p = orc.init(lif, 99) * np.float32(2.5)
    p[-4:] = orc.init(lif, 99)[-4:]
    ea = orc.entries(alif)
    pa = np.zeros(orc.param_count(alif), np.float32)
    el = {n: (o, s) for n, o, s in orc.entries(lif)}
    for n, o, s in ea:
        if n.endswith(".gamma"):
            pa[o:o + s] = 1.0
        else:
            lo, ls = el[n]
            pa[o:o + s] = p[lo:lo + ls]
    a = orc.forward_backward(alif, pa, pk, T, y, want_spikes=True)
    b = orc.forward_backward(lif, p, pk, T, y, want_spikes=True)
    assert a["loss"] == b["loss"]
    assert np.array_equal(a["spikes"][0], b["spikes"][0])
    for n, o, s in ea:
        if not n.endswith(".gamma"):
            lo, ls = el[n]
            assert np.array_equal(a["grads"][o:o + s], b["grads"][lo:lo + ls]), n


def test_rlif_entries_and_init(orc):
    net = Net(inp=10, hidden=(8, 6), classes=3, cell=("lif", "rlif"))
    e = orc.entries(net)
    assert [(n, sz) for n, _, sz in e] == [("l0.w", 80), ("l1.beta", 8), ("l2.w", 48), ("l3.beta", 6),
                                          ("l3.rec", 36), ("l4.w", 18), ("l5.beta", 3)]
    p = orc.init(net, 77)
    cell_key = orc.key_child(77, 3)
    _, o, s = e[4]
    assert np.array_equal(p[o:o + s], orc.truncated_normal(orc.key_child(cell_key, 4), 36, 0.0,
                                                          np.float32(1.0) / np.sqrt(np.float32(6))))


def test_rlif_zero_recurrence_is_lif(orc):
    """rec = 0 makes RLIF the reference LIF bit for bit (fb = 0 adds exactly)."""
    lif = Net(inp=30, hidden=(16,), classes=4)
    rl = Net(inp=30, hidden=(16,), classes=4, cell=("rlif",))
    B, T = 5, 25
    rng = np.random.default_rng(8)
    pk = orc.pack_time((rng.random((B, T, 30)) < 0.3).astype(np.uint8))
    y = rng.integers(0, 4, B).astype(np.int64)
    p = orc.init(lif, 5) * np.float32(2.5)
    el = {n: (o, s) for n, o, s in orc.entries(lif)}
    pr = np.zeros(orc.param_count(rl), np.float32)
    er = orc.entries(rl)
    for n, o, s in er:
        if n in el:
            lo, ls = el[n]
            pr[o:o + s] = p[lo:lo + ls]
    a = orc.forward_backward(rl, pr, pk, T, y, want_spikes=True)
    b = orc.forward_backward(lif, p, pk, T, y, want_spikes=True)
    assert a["loss"] == b["loss"]
    assert np.array_equal(a["spikes"][0], b["spikes"][0])
    for n, o, s in er:
        if n in el:
            lo, ls = el[n]
            assert np.array_equal(a["grads"][o:o + s], b["grads"][lo:lo + ls]), n
