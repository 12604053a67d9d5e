"""CPU checks of the arithmetic the CUDA kernels restate from the reference's
numpy/OpenBLAS dependencies (numpy 2.x float32 exp, OpenBLAS SkylakeX
sgemv_n / sdot).  Each test re-implements the DEVICE algorithm in numpy
(exact FMA emulation) and compares it with what numpy does on this host --
the same comparison tests/test_gpu_parity.py makes with the real kernels.
Run on the GPU box too: OpenBLAS and numpy pick their kernels at run time.
"""
import numpy as np
import pytest

f32 = np.float32


def fma32(a, b, c):
    """Exact float32 fma.  a*b is exact in float64; a*b + c rounded to f64
    then to f32 can double-round only when the f64 sum lands exactly on an f32
    midpoint -- those (rare) lanes are redone in exact rational arithmetic."""
    a, b, c = np.broadcast_arrays(np.asarray(a, np.float32), np.asarray(b, np.float32),
                                  np.asarray(c, np.float32))
    s = a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)
    r = s.astype(np.float32)
    with np.errstate(invalid="ignore", over="ignore"):
        nb = np.nextafter(r, np.where(s > r.astype(np.float64), np.float32(np.inf),
                                      np.float32(-np.inf)).astype(np.float32))
        mid = (r.astype(np.float64) + nb.astype(np.float64)) / 2
    sus = np.nonzero(np.atleast_1d(s == mid))[0]
    if sus.size:
        from fractions import Fraction
        r = np.atleast_1d(r).copy()
        af, bf, cf = (np.atleast_1d(v) for v in (a, b, c))
        for i in sus:
            ex = Fraction(float(af[i])) * Fraction(float(bf[i])) + Fraction(float(cf[i]))
            cand = np.float32(float(ex))
            opts = (np.nextafter(cand, np.float32(-np.inf)), cand, np.nextafter(cand, np.float32(np.inf)))
            r[i] = min(opts, key=lambda x: (abs(Fraction(float(x)) - ex),
                                            int(np.float32(x).view(np.uint32)) & 1))
        r = r.reshape(a.shape)
    return r


def np_exp_port(x):
    """csrc/spx_common.cuh np_expf, restated."""
    x = np.asarray(x, np.float32)
    u = lambda h: np.uint32(h).view(np.float32)  # noqa: E731
    q = (x * u(0x3fb8aa3b)).astype(f32)
    q = ((q + f32(12582912.0)).astype(f32) - f32(12582912.0)).astype(f32)
    r = fma32(q, u(0xbf317200), x)
    r = fma32(q, u(0xb5bfbe8e), r)
    num = fma32(u(0x3a053dd8), r, u(0x3bdd7159))
    for c in (0x3d517d8c, 0x3e7d4c58, 0x3f39cbd5):
        num = fma32(num, r, u(c))
    num = fma32(num, r, f32(1.0))
    den = fma32(u(0x3cb0e832), r, u(0xbe8c6857))
    den = fma32(den, r, f32(1.0))
    out = np.ldexp((num / den).astype(f32), q.astype(np.int32)).astype(f32)
    out = np.where(x >= u(0x42b17218), np.float32(np.inf), out)
    out = np.where(x <= u(0xc2cff1b5), np.float32(0), out)
    return out


def test_np_exp_port_matches_numpy():
    r = np.random.default_rng(0)
    x = np.concatenate([r.uniform(-104, 0, 400_000), r.uniform(-5, 0, 200_000),
                        r.uniform(-1e-3, 0, 50_000), [0.0, -0.0, -87.33, -88.0, -103.9, -103.98,
                                                      -104.0, -150.0]]).astype(np.float32)
    with np.errstate(over="ignore", under="ignore"):
        ref = np.exp(x)
        got = np_exp_port(x)
    bad = np.nonzero(ref.view(np.uint32) != got.view(np.uint32))[0]
    assert bad.size == 0, (x[bad[:5]], ref[bad[:5]], got[bad[:5]])


def sgemv_z1(f, W):
    """Device z1 order (csrc/spx_predictor.cu mlp_and_decide)."""
    n, H = W.shape
    if n <= 48:
        acc = np.zeros(H, f32)
        for i in range(n):
            acc = fma32(np.full(H, f[i], f32), W[i], acc)
        return acc
    y = np.zeros(H, f32)
    i = 0
    for bs in (8, 4, 2, 1):
        while n - i >= bs:
            t = np.zeros(H, f32)
            for q in range(bs):
                t = fma32(np.full(H, f[i + q], f32), W[i + q], t)
            y = (y + t).astype(f32)
            i += bs
            if bs != 8:
                break
    return y


def sdot_z2(h, w):
    """Device z2 order (OpenBLAS SkylakeX sdot)."""
    H = h.size
    n1 = H & ~31
    n64 = n1 & ~63
    dot = f32(0)
    if n1:
        A = np.zeros((4, 16), f32)
        for b in range(0, n64, 64):
            for a in range(4):
                A[a] = fma32(h[b + 16 * a:b + 16 * a + 16], w[b + 16 * a:b + 16 * a + 16], A[a])
        acc = (A[:, :8] + A[:, 8:]).astype(f32)
        if n1 > n64:
            for a in range(4):
                s = n64 + 8 * a
                acc[a] = fma32(h[s:s + 8], w[s:s + 8], acc[a])
        s = (((acc[0] + acc[1]).astype(f32) + acc[2]).astype(f32) + acc[3]).astype(f32)
        hh = (s[:4] + s[4:]).astype(f32)
        dot = f32(f32(hh[0] + hh[1]) + f32(hh[2] + hh[3]))
    for i in range(n1, H):
        dot = f32(dot + f32(h[i] * w[i]))
    return dot


@pytest.mark.parametrize("K", [1, 2, 4, 8, 16, 17, 20, 32, 64])
def test_mlp_hidden_layer_order(K):
    r = np.random.default_rng(K)
    H = 512
    for _ in range(4):
        f = r.standard_normal(3 * K).astype(f32)
        W = (r.standard_normal((3 * K, H)) * 0.1).astype(f32)
        assert np.array_equal((f @ W).view(np.uint32), sgemv_z1(f, W).view(np.uint32))


@pytest.mark.parametrize("H", [32, 64, 96, 128, 512, 1024])
def test_mlp_output_dot_order(H):
    r = np.random.default_rng(H)
    for _ in range(50):
        h = np.maximum(r.standard_normal(H), 0).astype(f32)
        w = r.standard_normal(H).astype(f32)
        assert (h @ w).view(np.uint32) == sdot_z2(h, w).view(np.uint32)


def test_z_cut_is_the_exact_decision_boundary():
    from paper_2504_08850_b200.predictor import _sigmoid64, z_cut
    for thr in (0.5, 0.7, 0.3, 0.999, 1e-6, 0.9999999):
        c = np.float32(z_cut(thr))
        below = np.nextafter(c, np.float32(-np.inf))
        assert _sigmoid64(np.float64(c)) > thr
        assert not (_sigmoid64(np.float64(below)) > thr)
        # monotone in a window around the cut
        bits = c.view(np.int32) + np.arange(-1000, 1000, dtype=np.int32)
        zs = bits.view(np.float32) if c > 0 else None
        if zs is not None:
            dec = _sigmoid64(zs.astype(np.float64)) > thr
            assert np.all(dec == (zs >= c))
    # thr 0.5: sigmoid(1e-16) > 0.5 is False, sigmoid(2e-16) > 0.5 is True
    assert 1e-16 < z_cut(0.5) <= 2e-16
    assert np.isnan(z_cut(1.0)) and z_cut(-0.5) == float("-inf")
