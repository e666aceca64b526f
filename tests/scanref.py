"""numpy float32 restatement of the LIF forward/backward scans (test helper).

Same operation order as neuron.hpp:127-136 and the tape closures, so that
given the GPU's own projection I (or dS), the GPU scan outputs must match
these BIT FOR BIT.  Used only by tests.
"""
import numpy as np

F = np.float32
PI_F = F(np.pi)


def clip01(b):
    lo = np.where(F(0) < b, b, F(0)).astype(F)
    return np.where(lo < F(1), lo, F(1)).astype(F)


def surrogate(act, k, aux, x):
    k = F(k)
    if act == "superspike":
        d = F(1) + k * np.abs(x)
        return (F(1) / (d * d)).astype(F)
    if act == "triangular":
        r = F(1) - np.abs(k * x)
        return np.where(F(0) < r, r, F(0)).astype(F)
    if act == "arctan":
        u = PI_F * k * x / F(2)
        return (F(1) / (F(1) + u * u)).astype(F)
    if act == "sigmoid":  # declared (oracle/spiketrain_oracle.h): k e / (1 + e)^2, e = exp(-k|x|)
        e = np.exp(-(k * np.abs(x))).astype(F)
        d = (F(1) + e).astype(F)
        return ((k * e) / (d * d)).astype(F)
    if act == "boxcar":
        return np.where(np.abs(x) <= k / F(2), F(aux), F(0)).astype(F)
    return np.ones_like(x, dtype=F)


def lif_forward(I, beta, theta):
    """I [B,T,H] f32 -> (V entering each step, spikes u8)."""
    B, T, H = I.shape
    vb = clip01(beta.astype(F))
    theta = F(theta)
    v = np.zeros((B, H), F)
    V = np.empty_like(I)
    S = np.empty(I.shape, np.uint8)
    for t in range(T):
        V[:, t] = v
        pre = v + (-theta)
        s = (pre >= F(0))
        m = v * vb
        a = m + I[:, t]
        r = s.astype(F) * theta
        v = (a - r).astype(F)
        S[:, t] = s
    return V, S


def lif_backward(dS, V, beta, theta, act, k, aux):
    """dS, V [B,T,H] -> dI [B,T,H], per-neuron dbeta (before clip mask, summed)."""
    B, T, H = dS.shape
    vb = clip01(beta.astype(F))
    theta = F(theta)
    G = np.zeros((B, H), F)
    dI = np.empty_like(dS)
    for t in range(T - 1, -1, -1):
        dI[:, t] = G
        rg = -G
        gs = dS[:, t] + rg * theta
        pre = V[:, t] + (-theta)
        gpre = gs * surrogate(act, k, aux, pre)
        G = (G * vb + gpre).astype(F)
    return dI


def alif_forward(I, beta, gamma, theta):
    """Declared ALIF cell (oracle/spiketrain_oracle.h), same op order:
    I [B,T,H] f32 -> (V, a entering each step, spikes u8)."""
    B, T, H = I.shape
    vb = clip01(beta.astype(F))
    gc = clip01(gamma.astype(F))
    omg = (F(1) - gc).astype(F)
    theta = F(theta)
    v = np.zeros((B, H), F)
    a = np.zeros((B, H), F)
    V = np.empty_like(I)
    A = np.empty_like(I)
    S = np.empty(I.shape, np.uint8)
    for t in range(T):
        V[:, t] = v
        A[:, t] = a
        th = (theta + a).astype(F)
        pre = (v - th).astype(F)
        s = pre >= F(0)
        ai = (v * vb + I[:, t]).astype(F)
        v = (ai - s.astype(F) * th).astype(F)
        a = (a * gc + omg * s.astype(F)).astype(F)
        S[:, t] = s
    return V, A, S


def rlif_forward(I, beta, rec, theta):
    """Declared RLIF cell (oracle/spiketrain_oracle.h), same op order: fb sums the
    rows of rec [H][H] of the spiking neurons in ascending order.
    I [B,T,H] f32 -> (V entering each step, spikes u8)."""
    B, T, H = I.shape
    vb = clip01(beta.astype(F))
    theta = F(theta)
    rec = rec.reshape(H, H).astype(F)
    v = np.zeros((B, H), F)
    V = np.empty_like(I)
    S = np.empty(I.shape, np.uint8)
    zero = np.zeros((B, H), F)
    for t in range(T):
        V[:, t] = v
        s = (v + (-theta)) >= F(0)
        fb = np.zeros((B, H), F)
        for i in np.nonzero(s.any(axis=0))[0]:
            fb = (fb + np.where(s[:, i:i + 1], rec[i][None, :], zero)).astype(F)
        ai = (v * vb + I[:, t]).astype(F)
        v = ((ai + fb).astype(F) - s.astype(F) * theta).astype(F)
        S[:, t] = s
    return V, S
