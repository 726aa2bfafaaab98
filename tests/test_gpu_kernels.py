"""Kernel-level parity on the B200: every C-ABI entry point against its CPU oracle.

Bars: bit-exact for the noise bitstream (fp32 rounding of numpy's fp64
draws); fp32 tolerances (stated per test) for floating-point kernels.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _cpu(t):
    return t.double().cpu().numpy()


# ---------------------------------------------------------------- noise (K1+K2)
@pytest.mark.parametrize("seed,prefix,t,ch,N,rows,cols", [
    (0, (), 1, 0, 5, 2, 3),
    (3, (), 2, 1, 37, 5, 7),
    (12345, (7, 2), 4, 2, 16, 8, 33),
    (2 ** 40 + 5, (1,), 0, 3, 9, 1, 1),
])
def test_noise_bit_exact_vs_numpy(dev_ops, seed, prefix, t, ch, N, rows, cols):
    from oracle import noise as onoise
    from paper_2410_09663_b200.matvar import entropy_head

    ref = onoise.member_normals(seed, prefix, t, ch, N, (rows, cols), backend="numpy")
    out = dev_ops.zeros(rows, N * cols)
    dev_ops.noise_fill(entropy_head(seed, prefix), t, ch, 0, N, rows, cols, out=out)
    got = out.cpu().numpy().reshape(rows, N, cols).transpose(1, 0, 2)
    assert np.array_equal(got, ref.astype(np.float32))


@pytest.mark.parametrize("cols", [66, 64])
def test_noise_bit_exact_many_streams_with_tail(dev_ops, cols):
    """~270k normals: exercises the wedge (0.8%) and tail (0.02%) rejection paths
    (cols 66: direct stores; cols 64: row-staged float4 path)."""
    from oracle import noise as onoise
    from paper_2410_09663_b200.matvar import entropy_head

    N, rows = 64, 64
    ref = onoise.member_normals(9, (), 5, 1, N, (rows, cols), backend="c")
    assert np.abs(ref).max() > 3.6541528853610088  # at least one tail sample present
    out = dev_ops.zeros(rows, N * cols)
    dev_ops.noise_fill(entropy_head(9, ()), 5, 1, 0, N, rows, cols, out=out)
    got = out.cpu().numpy().reshape(rows, N, cols).transpose(1, 0, 2)
    assert np.array_equal(got, ref.astype(np.float32))


@pytest.mark.parametrize("N,rows,cols,m0", [(6, 4, 5, 11), (6, 4, 32, 11), (5, 9, 128, 3),
                                            (3, 70, 512, 0)])
def test_noise_member_offset_diag_and_base(dev_ops, N, rows, cols, m0):
    from oracle import noise as onoise
    from paper_2410_09663_b200.matvar import entropy_head

    diag = np.linspace(0.5, 3.0, rows)
    ref = onoise.member_normals(1, (), 3, 2, m0 + N, (rows, cols), backend="c")[m0:]
    col = (diag[None, :, None] * ref).astype(np.float32)
    base = torch.randn(rows, N * cols, device=dev_ops.device)
    out = dev_ops.zeros(rows, N * cols)
    plus = dev_ops.zeros(rows, N * cols)
    dev_ops.noise_fill(entropy_head(1, ()), 3, 2, m0, N, rows, cols,
                       diag=dev_ops.to_device(diag, dtype=torch.float64), out=out, base=base,
                       out_plus=plus)
    got = out.cpu().numpy().reshape(rows, N, cols).transpose(1, 0, 2)
    assert np.array_equal(got, col)
    exp_plus = base.cpu().numpy() + col.transpose(1, 0, 2).reshape(rows, -1)
    assert np.array_equal(plus.cpu().numpy(), exp_plus.astype(np.float32))


# ---------------------------------------------------------------- member statistics (K4/K5)
@pytest.mark.parametrize("rows,N,cols", [(3, 4, 5), (40, 100, 32), (7, 1000, 3)])
def test_member_stats(dev_ops, rows, N, cols):
    rng = np.random.default_rng(rows)
    x = rng.standard_normal((rows, N, cols)).astype(np.float32) + 3.0
    src = dev_ops.to_device(x.reshape(rows, -1))
    acc = dev_ops.zeros(rows, cols, dtype=torch.float64)
    dev_ops.member_sum(src, N, cols, None, acc)
    mean = dev_ops.zeros(rows, cols)
    anom = dev_ops.zeros(rows, N * cols)
    dev_ops.member_center(src, N, cols, None, acc, N, mean=mean, anom=anom)
    x64 = x.astype(np.float64)
    np.testing.assert_allclose(_cpu(mean), x64.mean(axis=1), rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(_cpu(anom).reshape(rows, N, cols), x64 - x64.mean(axis=1, keepdims=True),
                               rtol=1e-5, atol=1e-5)


def test_member_stats_identical_members_exact_zero(dev_ops):
    """Shift by member 0: identical members give exactly zero anomalies at any N."""
    rng = np.random.default_rng(0)
    one = rng.standard_normal((6, 1, 7)).astype(np.float32)
    x = np.repeat(one, 100, axis=1)
    src = dev_ops.to_device(x.reshape(6, -1))
    acc = dev_ops.zeros(6, 7, dtype=torch.float64)
    dev_ops.member_sum(src, 100, 7, None, acc)
    mean, anom = dev_ops.zeros(6, 7), dev_ops.zeros(6, 700)
    dev_ops.member_center(src, 100, 7, None, acc, 100, mean=mean, anom=anom)
    assert np.array_equal(mean.cpu().numpy(), one[:, 0, :])
    assert not anom.cpu().numpy().any()


# ---------------------------------------------------------------- GEMM
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("M,N,K,split", [(5, 7, 3, 1), (130, 257, 300, 1), (300, 140, 5000, 7),
                                         (64, 64, 0, 1)])
def test_gemm_simt(dev_ops, ta, tb, M, N, K, split):
    g = torch.Generator().manual_seed(M * 7 + N)
    A = torch.randn(K, M, generator=g) if ta else torch.randn(M, K, generator=g)
    B = torch.randn(N, K, generator=g) if tb else torch.randn(K, N, generator=g)
    C0 = torch.randn(M, N, generator=g)
    bias = torch.randn(M, 4, generator=g)
    C = dev_ops.zeros(M, N)
    dev_ops.gemm(A.to(dev_ops.device), B.to(dev_ops.device), C, trans_a=ta, trans_b=tb,
                 alpha=0.7, beta=-1.5, C0=C0.to(dev_ops.device), bias=bias.to(dev_ops.device),
                 bias_cols=4, split=split, engine=1)
    exp = 0.7 * ((A.t() if ta else A).double() @ (B.t() if tb else B).double()) - 1.5 * C0.double()
    exp = exp + bias.double()[:, [c % 4 for c in range(N)]]
    err = (C.double().cpu() - exp).abs().max().item()
    assert err <= 2e-6 * max(1.0, K ** 0.5) * 10, err


def test_gemm_triangular_skip(dev_ops):
    """tri_rows/tri_k: rows of block s start at k = s * tri_k (block upper-triangular A)."""
    d, p, S = 6, 4, 5
    A = torch.randn(S * d, S * p)
    for s in range(S):
        A[s * d:(s + 1) * d, :s * p] = 0.0
    B = torch.randn(S * p, 9)
    C = dev_ops.zeros(S * d, 9)
    dev_ops.gemm(A.to(dev_ops.device), B.to(dev_ops.device), C, tri=(d, p), engine=1)
    np.testing.assert_allclose(C.double().cpu().numpy(), (A.double() @ B.double()).numpy(),
                               rtol=1e-5, atol=1e-5)


# ---------------------------------------------------------------- gain solve (K8)
@pytest.mark.parametrize("p", [1, 6, 64, 256])
def test_spd_inverse(dev_ops, p):
    rng = np.random.default_rng(p)
    a = rng.standard_normal((p, p + 3))
    s = (a @ a.T / (p + 3) + 0.5 * np.eye(p)).astype(np.float32)
    s[0, -1] += 1e-3  # asymmetry is symmetrized away
    inv = dev_ops.zeros(p, p)
    st, jit = dev_ops.zeros(1, dtype=torch.int32), dev_ops.zeros(1, dtype=torch.int32)
    dev_ops.spd_inverse(dev_ops.to_device(s), 2.0, inv, st, jit)
    sym = 2.0 * 0.5 * (s.astype(np.float64) + s.T.astype(np.float64))
    ref = np.linalg.inv(sym)
    assert st.item() == 0 and jit.item() == 0
    np.testing.assert_allclose(_cpu(inv), ref, rtol=2e-4, atol=2e-4 * np.abs(ref).max())


def test_spd_inverse_jitter_and_failure(dev_ops):
    p = 5
    st, jit = dev_ops.zeros(1, dtype=torch.int32), dev_ops.zeros(1, dtype=torch.int32)
    inv = dev_ops.zeros(p, p)
    # zero matrix -> jitter 1e-30 -> inverse 1e30 I (the reference's degenerate path)
    dev_ops.spd_inverse(dev_ops.zeros(p, p), 1.0, inv, st, jit)
    assert st.item() == 0 and jit.item() == 1
    np.testing.assert_allclose(_cpu(inv), 1e30 * np.eye(p), rtol=1e-5)
    # indefinite even after jitter -> status 1 (reference raises LinAlgError)
    bad = -np.eye(p, dtype=np.float32)
    dev_ops.spd_inverse(dev_ops.to_device(bad), 1.0, inv, st, jit)
    assert st.item() == 1 and jit.item() == 2


# ---------------------------------------------------------------- CNN forecast (K3)
@pytest.mark.parametrize("n,widths,N", [(16, (2, 8, 1), 3), (32, (2, 16, 16, 1), 5),
                                        (40, (2, 32, 32, 1), 2), (128, (2, 32, 32, 1), 2),
                                        (40, (2, 32, 32, 32, 32, 32, 1), 2),  # C4 depth, weights in L1
                                        # deep tcgen05 path (cnn_deep.cu): 128 / 256-wide fields
                                        (256, (2, 32, 32, 32, 32, 32, 1), 2),
                                        (128, (2, 32, 32, 32, 1), 3),
                                        (256, (2, 32, 32, 1), 2)])
def test_cnn_forward(dev_ops, pm, n, widths, N):
    from oracle.models import cnn_step
    from paper_2410_09663_b200.engine import Forecaster

    model = pm.dynamics.CNNDynamics(rows=n, cols=n, widths=widths, seed=1)
    rng = np.random.default_rng(n)
    x = rng.standard_normal((N, n, n))
    u = rng.standard_normal((N, n, n))
    ref = cnn_step(x, u, model.weights, model.biases, model.alpha)
    last = dev_ops.to_device(np.concatenate([x, u], axis=1).transpose(1, 0, 2).reshape(2 * n, -1))
    out = dev_ops.zeros(n, N * n)
    fc = Forecaster(model, dev_ops, n, n)
    fc(dev_ops, last, out, n, N)
    got = _cpu(out).reshape(n, N, n).transpose(1, 0, 2)
    np.testing.assert_allclose(got, ref, rtol=1e-5, atol=2e-6)


# ---------------------------------------------------------------- tcgen05 3xTF32 contraction
@pytest.mark.parametrize("M,N,K,split", [(128, 256, 4096, 1), (300, 256, 131072, 0), (77, 6, 1000, 0),
                                         (1000, 100, 20000, 3), (640, 256, 131072, 0),
                                         (5, 32, 128, 1)])
def test_gemm_nt_tc_3xtf32(dev_ops, M, N, K, split):
    """Within fp32-FFMA accuracy of the fp64 product (1xTF32 would be ~1e-3 relative)."""
    g = torch.Generator().manual_seed(M + N + K)
    A = torch.randn(M, K, generator=g) + 0.5
    B = torch.randn(N, K, generator=g)
    dA, dB = A.to(dev_ops.device), B.to(dev_ops.device)
    bh, bl = dev_ops.empty(N, K), dev_ops.empty(N, K)
    dev_ops.tf32_split(dB, bh, bl)
    assert torch.equal((bh + bl).cpu(), B)
    C = dev_ops.zeros(M, N)
    dev_ops.gemm_nt_tc(dA, bh, bl, C, alpha=0.5, split=split)
    ref = 0.5 * (A.double() @ B.double().t())
    scale = 0.5 * (A.double().abs() @ B.double().abs().t())
    err = ((C.double().cpu() - ref).abs() / scale).max().item()
    # the SIMT FFMA engine on the same inputs: the fp32-accumulation error to match
    C2 = dev_ops.zeros(M, N)
    dev_ops.gemm(dA, dB, C2, trans_b=True, alpha=0.5, engine=1)
    err2 = ((C2.double().cpu() - ref).abs() / scale).max().item()
    assert err < 1e-5, err
    assert err < max(3 * err2, 1e-6), (err, err2)


@pytest.mark.parametrize("rows,cols,N", [(128, 128, 3), (40, 128, 5), (64, 64, 3), (64, 64, 8),
                                         (32, 32, 5), (20, 32, 4), (17, 64, 1)])
def test_cnn_forward_tcgen05_vs_oracle(dev_ops, pm, rows, cols, N):
    """The fused tcgen05 conv (widths 2-32-32-1) against the fp64 oracle; 32- and 64-wide
    fields pack 4 / 2 images per 128-pixel MMA row (odd N leaves padding columns)."""
    from oracle.models import cnn_step
    from paper_2410_09663_b200.engine import Forecaster

    model = pm.dynamics.CNNDynamics(rows=rows, cols=cols, widths=(2, 32, 32, 1), seed=3)
    model.state_rows = model.input_rows = rows
    rng = np.random.default_rng(rows)
    x = rng.standard_normal((N, rows, cols))
    u = rng.standard_normal((N, rows, cols))
    ref = cnn_step(x, u, model.weights, model.biases, model.alpha)
    last = dev_ops.to_device(np.concatenate([x, u], axis=1).transpose(1, 0, 2).reshape(2 * rows, -1))
    full = dev_ops.zeros(rows, N * cols + 64)
    full.fill_(7.0)  # sentinel: the padding columns of a partly filled MMA row are never written
    out = full[:, :N * cols]
    Forecaster(model, dev_ops, rows, rows)(dev_ops, last, out, rows, N)
    assert bool((full[:, N * cols:] == 7.0).all())
    got = _cpu(out).reshape(rows, N, cols).transpose(1, 0, 2)
    np.testing.assert_allclose(got, ref, rtol=1e-5, atol=2e-6)


def test_cnn_forward_tcgen05_matches_simt_many_members(dev_ops, pm, monkeypatch):
    """Persistent CTAs over > 148 members: tcgen05 path == SIMT path to fp32 rounding."""
    from paper_2410_09663_b200.engine import Forecaster

    n, N = 128, 300
    model = pm.dynamics.CNNDynamics(rows=n, cols=n, widths=(2, 32, 32, 1), seed=4)
    g = torch.Generator().manual_seed(0)
    last = torch.randn(2 * n, N * n, generator=g).to(dev_ops.device)
    fc = Forecaster(model, dev_ops, n, n)
    out_tc = dev_ops.zeros(n, N * n)
    fc(dev_ops, last, out_tc, n, N)
    monkeypatch.setenv("ENKS_CNN_TC", "0")
    out_simt = dev_ops.zeros(n, N * n)
    fc(dev_ops, last, out_simt, n, N)
    torch.cuda.synchronize()
    diff = (out_tc - out_simt).abs().max().item()
    assert diff < 2e-5, diff


@pytest.mark.parametrize("p", [33, 100, 288])
def test_spd_inverse_blocked_sizes(dev_ops, p):
    """Tile padding (p not a multiple of 32) and the largest supported p."""
    rng = np.random.default_rng(p + 1)
    a = rng.standard_normal((p, 2 * p))
    s = (a @ a.T / (2 * p) + 0.2 * np.eye(p)).astype(np.float32)
    inv = dev_ops.zeros(p, p)
    st, jit = dev_ops.zeros(1, dtype=torch.int32), dev_ops.zeros(1, dtype=torch.int32)
    dev_ops.spd_inverse(dev_ops.to_device(s), 1.0, inv, st, jit)
    ref = np.linalg.inv(s.astype(np.float64))
    assert st.item() == 0 and jit.item() == 0
    np.testing.assert_allclose(_cpu(inv), ref, rtol=2e-4, atol=2e-4 * np.abs(ref).max())


def test_fused_noise_multi_matches_single(dev_ops):
    """One launch for (W, V_X, V_U) == three enks_noise_fill launches, bit for bit."""
    from paper_2410_09663_b200.matvar import entropy_head

    N, cols, rows = 9, 6, (3, 5, 3)
    head = entropy_head(4, (1,))
    diag = [dev_ops.to_device(np.linspace(0.5, 2.0, r), dtype=torch.float64) for r in rows]
    base = [torch.randn(r, N * cols, device=dev_ops.device) for r in rows]
    single = [dev_ops.zeros(r, N * cols) for r in rows]
    plus1 = [dev_ops.zeros(r, N * cols) for r in rows]
    for k, r in enumerate(rows):
        dev_ops.noise_fill(head, 7, k, 0, N, r, cols, diag=diag[k], out=single[k], base=base[k],
                           out_plus=plus1[k])
    multi = [dev_ops.zeros(r, N * cols) for r in rows]
    plus2 = [dev_ops.zeros(r, N * cols) for r in rows]
    dev_ops.noise_fill_multi(head, 0, N, cols, [dict(t=7, ch=k, rows=r, diag=diag[k], out=multi[k],
                                                     base=base[k], out_plus=plus2[k])
                                                for k, r in enumerate(rows)])
    for k in range(3):
        assert torch.equal(single[k], multi[k]) and torch.equal(plus1[k], plus2[k])


@pytest.mark.parametrize("M,N,K,tri,split", [(256, 4096, 256, None, 1), (300, 256, 2000, None, 0),
                                             (77, 6, 40, None, 1), (1000, 100, 700, (200, 100), 1),
                                             (130, 130, 3000, None, 4), (256, 131072, 256, None, 1)])
def test_gemm_tc_general(dev_ops, M, N, K, tri, split):
    """C = alpha A B + beta C0 + bias via transposed split planes; triangular skip; N tiling."""
    g = torch.Generator().manual_seed(M + 3 * N + K)
    A = torch.randn(M, K, generator=g)
    if tri:
        d, p = tri
        for s in range(M // d + 1):
            A[s * d:(s + 1) * d, :min(K, s * p)] = 0.0
    B = torch.randn(K, N, generator=g)
    C0 = torch.randn(M, N, generator=g)
    bias = torch.randn(M, 4, generator=g)
    dA, dB = A.to(dev_ops.device), B.to(dev_ops.device)
    bh, bl = dev_ops.empty(N, K), dev_ops.empty(N, K)
    dev_ops.tf32_split(dB, bh, bl, transpose=True)
    assert torch.equal((bh + bl).cpu(), B.t())
    C = dev_ops.zeros(M, N)
    dev_ops.gemm_tc(dA, bh, bl, C, alpha=-0.5, beta=1.0, C0=C0.to(dev_ops.device),
                    bias=bias.to(dev_ops.device), bias_cols=4, tri=tri or (0, 0), split=split)
    ref = -0.5 * (A.double() @ B.double()) + C0.double() + bias.double()[:, [c % 4 for c in range(N)]]
    scale = 0.5 * (A.double().abs() @ B.double().abs()) + C0.double().abs() + 1.0
    err = ((C.double().cpu() - ref).abs() / scale).max().item()
    assert err < 1e-6, err


@pytest.mark.parametrize("M,N,K", [(128, 256, 4096), (300, 256, 131072), (77, 6, 1000), (640, 256, 8192),
                                   (5, 32, 64)])
def test_gemm_f16pair(dev_ops, M, N, K):
    """fp16-pair storage + kind::f16 contraction: fp32-FFMA-level accuracy (~2^-22 per product)."""
    g = torch.Generator().manual_seed(M + N + K)
    A = (torch.randn(M, K, generator=g) + 0.5) * torch.logspace(-3, 3, M).unsqueeze(1)
    B = torch.randn(N, K, generator=g)
    dA, dB = A.to(dev_ops.device), B.to(dev_ops.device)
    ah = torch.empty(M, K, dtype=torch.float16, device=dev_ops.device)
    al = torch.empty_like(ah)
    bh = torch.empty(N, K, dtype=torch.float16, device=dev_ops.device)
    bl = torch.empty_like(bh)
    sa, sb = dev_ops.empty(M), dev_ops.empty(N)
    dev_ops.f16pair_split(dA, ah, al, sa)
    dev_ops.f16pair_split(dB, bh, bl, sb)
    rec = dev_ops.empty(M, K)
    dev_ops.f16pair_recon(ah, al, sa, rec)
    assert ((rec.double().cpu() - A.double()).abs() / A.double().abs().amax(1, keepdim=True)).max() < 2e-7
    C = dev_ops.zeros(M, N)
    dev_ops.gemm_f16pair(ah, al, sa, bh, bl, sb, C, alpha=0.5)
    ref = 0.5 * (A.double() @ B.double().t())
    scale = 0.5 * (A.double().abs() @ B.double().abs().t())
    err = ((C.double().cpu() - ref).abs() / scale).max().item()
    assert err < 1e-6, err


def _burgers_forecaster(dev_ops, pm, g, mode, substeps, dt=0.001):
    from paper_2410_09663_b200.engine import Forecaster

    model = pm.dynamics.BurgersDynamics(pm.dynamics.BurgersConfig(grid_n=g, control_mode=mode,
                                                                  substeps=substeps, dt=dt))
    return model, Forecaster(model, dev_ops, 2 * g, model.input_rows)


@pytest.mark.parametrize("g,mode,substeps,N", [(8, "boundary", 1, 5), (32, "pointwise", 3, 100),
                                               (32, "boundary", 4, 37), (64, "pointwise", 2, 9),
                                               (128, "boundary", 3, 3), (128, "pointwise", 1, 2)])
def test_burgers_forward_vs_oracle(dev_ops, pm, g, mode, substeps, N):
    """Fused shared-memory kernel (g <= 64) and per-substep global kernel (g = 128)."""
    from oracle.models import burgers_step

    model, fc = _burgers_forecaster(dev_ops, pm, g, mode, substeps)
    rng = np.random.default_rng(g + N)
    base = pm.dynamics.make_initial_field(model.cfg, 0).packed
    x = base[None] + 0.1 * rng.standard_normal((N, 2 * g, g))
    u = rng.standard_normal((N, model.input_rows, g))
    ref, vmax = burgers_step(x, u, g, model.cfg.nu, model.cfg.dt, mode, substeps)
    last = np.concatenate([x, u], axis=1).transpose(1, 0, 2).reshape(2 * g + u.shape[1], N * g)
    last_d = dev_ops.to_device(last)
    out = dev_ops.zeros(2 * g, N * g)
    fc(dev_ops, last_d, out, 2 * g, N)
    got = out.double().cpu().numpy().reshape(2 * g, N, g).transpose(1, 0, 2)
    assert np.abs(got - ref).max() < 1e-5 * np.abs(ref).max()
    assert abs(float(fc.vmax[0]) - vmax) <= 1e-6 * vmax
    fc.check_cfl()


def test_burgers_cfl_and_nonfinite_flags(dev_ops, pm):
    from paper_2410_09663_b200.dynamics import CflError

    g, N = 16, 4
    _, fc = _burgers_forecaster(dev_ops, pm, g, "boundary", 1, dt=0.01)
    last = np.zeros((2 * g + 2, N * g))
    last[:2 * g] = 0.5                      # |phi| dt/dx = 0.5 * 0.01 * 15 = 0.075: fine
    out = dev_ops.zeros(2 * g, N * g)
    fc(dev_ops, dev_ops.to_device(last), out, 2 * g, N)
    fc.check_cfl()
    last[3, 5 * 1 + g] = 10.0               # 10 * 0.01 * 15 = 1.5 > 1 on member 1
    fc(dev_ops, dev_ops.to_device(last), out, 2 * g, N)
    with pytest.raises(CflError, match="CFL"):
        fc.check_cfl()
    _, fc = _burgers_forecaster(dev_ops, pm, g, "boundary", 1, dt=0.01)
    last[3, 5 + g] = np.nan
    fc(dev_ops, dev_ops.to_device(last), out, 2 * g, N)
    with pytest.raises(CflError, match="non-finite"):
        fc.check_cfl()
    with pytest.raises(CflError, match="nu"):
        _burgers_forecaster(dev_ops, pm, g, "boundary", 1, dt=0.5)


@pytest.mark.parametrize("M,N,K", [(600, 300, 1024), (77, 513, 4096)])
def test_gemm_nt_f16pair_blocked_columns(dev_ops, M, N, K):
    """Covariance-tracking contraction: fp16-pair planes, N > 256 in 256-column launches."""
    g = torch.Generator().manual_seed(M * N)
    A = torch.randn(M, K, generator=g)
    B = torch.randn(N, K, generator=g)
    C = dev_ops.zeros(M, N)
    dev_ops.gemm_nt_f16pair(A.to(dev_ops.device), B.to(dev_ops.device), C, alpha=0.25)
    ref = 0.25 * (A.double() @ B.double().t())
    scale = 0.25 * (A.double().abs() @ B.double().abs().t())
    assert ((C.double().cpu() - ref).abs() / scale).max().item() < 1e-6
    Cs = dev_ops.zeros(M, M)
    dA = A.to(dev_ops.device)
    dev_ops.gemm_nt_f16pair(dA, dA, Cs)
    refs = A.double() @ A.double().t()
    # Gram diagonals are all-positive sums: the tensor core's truncating TMEM accumulation
    # within one chain biases them (gemm_f16p.cu kF16pChainDefault: ~2.9e-6 at 16 chunks)
    assert ((Cs.double().cpu() - refs).abs() / (A.double().abs() @ A.double().abs().t())).max() < 5e-6


def test_f16pair_gram_diagonal_bias_at_c3_depth(dev_ops):
    """Sigma_y-like Gram matrix at C3's contraction depth (K = N m = 131072, p = 256, split-K as
    in the smoother): the one-sided truncation bias of the TMEM chains on the positive diagonal
    stays within the chain-length bound c (KC/16) 3 2^-25 x 2 (c = 16 chunks of KC = 32), and the
    signed error of the off-diagonal entries stays at fp32-sum level."""
    g = torch.Generator().manual_seed(11)
    p, K = 256, 131072
    Y = torch.randn(p, K, generator=g) * torch.logspace(-1, 1, p).unsqueeze(1)
    f16 = torch.float16
    yh, yl, yi = dev_ops.empty(p, K, dtype=f16), dev_ops.empty(p, K, dtype=f16), dev_ops.empty(p)
    dev_ops.f16pair_split(Y.to(dev_ops.device), yh, yl, yi)
    C = dev_ops.zeros(p, p)
    dev_ops.gemm_f16pair(yh, yl, yi, yh, yl, yi, C)
    Yd = Y.double()
    ref = Yd @ Yd.t()
    diag_rel = ((C.double().cpu().diagonal() - ref.diagonal()) / ref.diagonal())
    bound = 2 * 16 * (32 / 16) * 3 * 2.0 ** -25
    print(f"diag rel bias mean {diag_rel.mean().item():.2e} min {diag_rel.min().item():.2e} "
          f"bound {bound:.2e}")
    assert diag_rel.abs().max().item() < bound
    scale = (Yd.abs() @ Yd.abs().t())
    off = ((C.double().cpu() - ref).abs() / scale)
    off.fill_diagonal_(0)
    assert off.max().item() < 1e-6


@pytest.mark.parametrize("p,q,K", [(256, 256, 4096 + 128), (256, 200, 1000), (128, 96, 776)])
def test_gemm_f16pair_ex_shift_operands(dev_ops, p, q, K):
    """Newest-slice shift: transposed re-split of fp16-pair rows, then the fused-epilogue GEMM
    C = C0 + bias - G Yc with N = K in 256-column tiles (the coalesced transposed epilogue; rows
    and columns not multiples of the 128 x 256 tile)."""
    g = torch.Generator().manual_seed(5 + q)
    m = 128
    Y = torch.randn(p, K, generator=g) * torch.logspace(-2, 2, p).unsqueeze(1)
    G = torch.randn(q, p, generator=g) * 0.01
    C0 = torch.randn(q, K, generator=g)
    bias = torch.randn(q, m, generator=g)
    f16 = torch.float16
    yh, yl = dev_ops.empty(p, K, dtype=f16), dev_ops.empty(p, K, dtype=f16)
    yi = dev_ops.empty(p)
    dev_ops.f16pair_split(Y.to(dev_ops.device), yh, yl, yi)
    th, tl, ti = dev_ops.empty(K, p, dtype=f16), dev_ops.empty(K, p, dtype=f16), dev_ops.empty(K)
    dev_ops.f16pair_transpose(yh, yl, yi, th, tl, ti)
    rec = dev_ops.empty(K, p)
    dev_ops.f16pair_recon(th, tl, ti, rec)
    assert ((rec.double().cpu() - Y.t().double()).abs() /
            Y.t().double().abs().amax(1, keepdim=True)).max() < 5e-7
    gh, gl, gi = dev_ops.empty(q, p, dtype=f16), dev_ops.empty(q, p, dtype=f16), dev_ops.empty(q)
    dev_ops.f16pair_split(G.to(dev_ops.device), gh, gl, gi)
    out = dev_ops.zeros(q, K)
    dev_ops.gemm_f16pair_ex(gh, gl, gi, th, tl, ti, out, alpha=-1.0, beta=1.0,
                            C0=C0.to(dev_ops.device), bias=bias.to(dev_ops.device), bias_cols=m)
    ref = C0.double() + bias.double()[:, [k % m for k in range(K)]] - G.double() @ Y.double()
    scale = (G.double().abs() @ Y.double().abs()) + C0.double().abs() + bias.double().abs().amax()
    assert ((out.double().cpu() - ref).abs() / scale).max().item() < 1e-6


@pytest.mark.parametrize("p,q,K,m", [(256, 256, 4096 + 128, 128), (256, 200, 1000, 128),
                                     (128, 96, 776, 128), (256, 256, 96 * 40, 96)])
def test_gemm_f16pair_ex_mn_shift(dev_ops, p, q, K, m):
    """Newest-slice shift with B = the Yc basis rows themselves (MN-major, K x N): G_tt takes Yc's
    per-row scale before its split (enks_f16pair_split_cs), no transposed planes.  The cases cover
    the shared-memory-staged epilogue (full 32-row x 128-column blocks) and its row-per-thread
    fallback (ragged rows / columns, bias period m = 96 not a multiple of the 128-column block)."""
    g = torch.Generator().manual_seed(7 + q + m)
    Y = torch.randn(p, K, generator=g) * torch.logspace(-2, 2, p).unsqueeze(1)
    G = torch.randn(q, p, generator=g) * 0.01
    C0 = torch.randn(q, K, generator=g)
    bias = torch.randn(q, m, generator=g)
    f16 = torch.float16
    yh, yl = dev_ops.empty(p, K, dtype=f16), dev_ops.empty(p, K, dtype=f16)
    yi = dev_ops.empty(p)
    dev_ops.f16pair_split(Y.to(dev_ops.device), yh, yl, yi)
    gh, gl, gi = dev_ops.empty(q, p, dtype=f16), dev_ops.empty(q, p, dtype=f16), dev_ops.empty(q)
    dev_ops.f16pair_split_cs(G.to(dev_ops.device), yi, gh, gl, gi)
    out = dev_ops.zeros(q, K)
    dev_ops.gemm_f16pair_ex_mn(gh, gl, gi, yh, yl, out, alpha=-1.0, beta=1.0,
                               C0=C0.to(dev_ops.device), bias=bias.to(dev_ops.device), bias_cols=m)
    ref = C0.double() + bias.double()[:, [k % m for k in range(K)]] - G.double() @ Y.double()
    scale = (G.double().abs() @ Y.double().abs()) + C0.double().abs() + bias.double().abs().amax()
    assert ((out.double().cpu() - ref).abs() / scale).max().item() < 1e-6


@pytest.mark.parametrize("p", [289, 300, 512, 576])
def test_spd_inverse_schur_blocks(dev_ops, p):
    """p > 288: 2 x 2 Schur complement of two one-CTA factorisations."""
    rng = np.random.default_rng(p)
    a = rng.standard_normal((p, p + 7))
    s = (a @ a.T / (p + 7) + 0.5 * np.eye(p)).astype(np.float32)
    s[0, -1] += 1e-3
    inv = dev_ops.zeros(p, p)
    st, jit = dev_ops.zeros(1, dtype=torch.int32), dev_ops.zeros(1, dtype=torch.int32)
    dev_ops.spd_inverse(dev_ops.to_device(s), 0.5, inv, st, jit)
    sym = 0.5 * 0.5 * (s.astype(np.float64) + s.T.astype(np.float64))
    ref = np.linalg.inv(sym)
    assert st.item() == 0 and jit.item() == 0
    np.testing.assert_allclose(_cpu(inv), ref, rtol=2e-4, atol=2e-4 * np.abs(ref).max())


def test_spd_inverse_schur_jitter_and_failure(dev_ops):
    p = 400
    st, jit = dev_ops.zeros(1, dtype=torch.int32), dev_ops.zeros(1, dtype=torch.int32)
    inv = dev_ops.zeros(p, p)
    dev_ops.spd_inverse(dev_ops.zeros(p, p), 1.0, inv, st, jit)  # jitter 1e-30 path
    assert st.item() == 0 and jit.item() == 1
    np.testing.assert_allclose(_cpu(inv), 1e30 * np.eye(p), rtol=1e-5)
    # rank-deficient PSD (N < p): the reference's jitter makes it SPD
    a = np.random.default_rng(1).standard_normal((p, 50))
    st.zero_()
    jit.zero_()
    dev_ops.spd_inverse(dev_ops.to_device(a @ a.T), 1.0, inv, st, jit)
    assert jit.item() == 1
    # indefinite even after jitter -> status
    st.zero_()
    bad = -np.eye(p)
    dev_ops.spd_inverse(dev_ops.to_device(bad), 1.0, inv, st, jit)
    assert st.item() == 1 and np.isnan(_cpu(inv)).all()


def test_noise_bit_exact_two_million(dev_ops):
    """2M normals (~24k wedge tests, a few hundred tails): the single-precision screening of
    the wedge test must reproduce numpy's double-precision decisions exactly."""
    from oracle import noise as onoise
    from paper_2410_09663_b200.matvar import entropy_head

    N, rows, cols = 64, 64, 512
    ref = onoise.member_normals(21, (3,), 2, 0, N, (rows, cols), backend="c")
    out = dev_ops.zeros(rows, N * cols)
    dev_ops.noise_fill(entropy_head(21, (3,)), 2, 0, 0, N, rows, cols, out=out)
    got = out.cpu().numpy().reshape(rows, N, cols).transpose(1, 0, 2)
    assert np.array_equal(got, ref.astype(np.float32))


# ------------------------------------------------ derived-U chain and fused observation centring
@pytest.mark.parametrize("ns,n,l,m,p", [(1, 4, 3, 5, 6), (7, 16, 8, 32, 24), (50, 128, 128, 128, 256)])
def test_uchain_apply(dev_ops, ns, n, l, m, p):
    """enks_uchain_apply: X / dU mean increments, U rows by prefix sums over slices; newest-slice
    gain rows [X of the last slice; sum of the dU rows] (fp32, tolerance 1e-5 relative)."""
    g = torch.Generator(device="cuda").manual_seed(ns)
    ds, d = n + l, n + 2 * l
    delta = torch.randn(ns * ds, m, device="cuda", generator=g)
    mean = torch.randn(ns * d, m, device="cuda", generator=g)
    gcol = torch.randn(ns * ds, p, device="cuda", generator=g)
    gtt = torch.empty(n + l, p, device="cuda")
    ref_mean = mean.double().clone().view(ns, d, m)
    dc = delta.double().view(ns, ds, m)
    ref_mean[:, :n] += dc[:, :n]
    ref_mean[:, n + l:] += dc[:, n:]
    ref_mean[:, n:n + l] += torch.cumsum(dc[:, n:], dim=0)
    gc = gcol.double().view(ns, ds, p)
    ref_g = torch.cat([gc[-1, :n], gc[:, n:].sum(dim=0)])
    dev_ops.uchain_apply(delta, mean, gcol, gtt, ns, n, l, m, p)
    torch.cuda.synchronize()
    assert (mean.double().view(ns, d, m) - ref_mean).abs().max() <= 1e-5 * ref_mean.abs().max()
    assert (gtt.double() - ref_g).abs().max() <= 1e-5 * ref_g.abs().max()


@pytest.mark.parametrize("rows,N,cols", [(6, 8, 4), (256, 64, 128), (100, 33, 32)])
def test_member_center_f16pair_t_two_sources(dev_ops, rows, N, cols):
    """Two-source member sum + centring into pair rows and transposed pair planes: equals the
    centred (src + src2) of the fp32 path to the pair precision (2^-20 relative)."""
    g = torch.Generator(device="cuda").manual_seed(rows)
    K = N * cols
    src = torch.randn(rows, K, device="cuda", generator=g) + 3.0
    src2 = 0.1 * torch.randn(rows, K, device="cuda", generator=g)
    acc = torch.zeros(rows, cols, dtype=torch.float64, device="cuda")
    amax = torch.zeros(rows, cols, device="cuda")
    dev_ops.member_sum(src, N, cols, None, acc, amax, src2=src2)
    f16 = torch.float16
    h, lo, inv = (torch.empty(rows, K, dtype=f16, device="cuda"),
                  torch.empty(rows, K, dtype=f16, device="cuda"), torch.empty(rows, device="cuda"))
    ldt = rows + (rows & 1)
    th, tl, tinv = (torch.empty(K, ldt, dtype=f16, device="cuda"),
                    torch.empty(K, ldt, dtype=f16, device="cuda"), torch.empty(K, device="cuda"))
    mean = torch.empty(rows, cols, device="cuda")
    dev_ops.member_center_f16pair_t(src, src2, N, cols, None, acc, amax, N, mean, h, lo, inv,
                                    th[:, :rows], tl[:, :rows], tinv)
    torch.cuda.synchronize()
    y = (src + src2).double().view(rows, N, cols)
    mu = y.mean(dim=1)
    anom = (y - mu[:, None, :]).reshape(rows, K)
    scale = anom.abs().max()
    assert (mean.double() - mu).abs().max() <= 1e-6 * mu.abs().max()
    rec = (h.double() + lo.double()) * inv.double()[:, None]
    assert (rec - anom).abs().max() <= 2 ** -20 * scale
    rect = (th[:, :rows].double() + tl[:, :rows].double()) * tinv.double()[:, None]
    assert (rect - anom.t()).abs().max() <= 2 ** -20 * scale


def test_member_center_f16pair_skipped_rows(dev_ops):
    """Rows [skip0, skip1) (the U block under the derived-U chain) stay out of the basis; the
    other rows move up; the fp32 copy of the first rows_f32 rows keeps every row."""
    rows, N, cols, s0, s1 = 12, 16, 8, 4, 8
    g = torch.Generator(device="cuda").manual_seed(3)
    src = torch.randn(rows, N * cols, device="cuda", generator=g)
    acc = torch.zeros(rows, cols, dtype=torch.float64, device="cuda")
    amax = torch.zeros(rows, cols, device="cuda")
    dev_ops.member_sum(src, N, cols, None, acc, amax)
    f16 = torch.float16
    outs = {}
    for skip in ((0, 0), (s0, s1)):
        hr = rows - (skip[1] - skip[0])
        h, lo, inv = (torch.empty(hr, N * cols, dtype=f16, device="cuda"),
                      torch.empty(hr, N * cols, dtype=f16, device="cuda"),
                      torch.empty(hr, device="cuda"))
        f32 = torch.empty(rows, N * cols, device="cuda")
        mean = torch.empty(rows, cols, device="cuda")
        dev_ops.member_center_f16pair(src, N, cols, None, acc, amax, N, mean, h, lo, inv,
                                      f32=f32, rows_f32=rows, skip=skip)
        outs[skip] = (h, lo, inv, f32, mean)
    full, part = outs[(0, 0)], outs[(s0, s1)]
    keep = list(range(s0)) + list(range(s1, rows))
    for a, b in zip(full[:3], part[:3]):
        assert torch.equal(a[keep], b)
    assert torch.equal(full[3], part[3]) and torch.equal(full[4], part[4])


@pytest.mark.parametrize("cols,N", [(128, 37), (64, 20), (32, 9)])
def test_cnn_forward_noise_matches_separate_launches(dev_ops, pm, cols, N):
    """enks_cnn_forward_noise (noise drawn by the fused forecast's idle warps) == the forecast
    and enks_noise_fill_multi launched separately, bit for bit."""
    from paper_2410_09663_b200.engine import Forecaster
    from paper_2410_09663_b200.matvar import entropy_head

    n = cols
    model = pm.dynamics.CNNDynamics(rows=n, cols=cols, widths=(2, 32, 32, 1), seed=1)
    fc = Forecaster(model, dev_ops, n, n)
    assert dev_ops.cnn_noise_fusable(fc, n)
    K = N * cols
    g = torch.Generator(device="cuda").manual_seed(cols)
    last = torch.randn(2 * n, K, device="cuda", generator=g)
    diag = [torch.rand(n, dtype=torch.float64, device="cuda", generator=g) + 0.5 for _ in range(3)]
    head = entropy_head(4, (2,))
    outs = {}
    for fused in (False, True):
        o = dict(x=torch.empty(n, K, device="cuda"), w=torch.empty(n, K, device="cuda"),
                 u=torch.empty(n, K, device="cuda"), vx=torch.empty(n, K, device="cuda"),
                 vu=torch.empty(n, K, device="cuda"))
        jobs = [dict(t=3, ch=0, rows=n, diag=diag[0], out=o["w"], base=last[n:], out_plus=o["u"]),
                dict(t=3, ch=1, rows=n, diag=diag[1], out=o["vx"]),
                dict(t=3, ch=2, rows=n, diag=diag[2], out=o["vu"])]
        if fused:
            dev_ops.cnn_forward_noise(fc, last[:n], last[n:], o["x"], N, head, 5, jobs)
        else:
            dev_ops.noise_fill_multi(head, 5, N, cols, jobs)
            fc(dev_ops, last, o["x"], n, N)
        torch.cuda.synchronize()
        outs[fused] = o
    for k in outs[False]:
        assert torch.equal(outs[False][k], outs[True][k]), k


@pytest.mark.parametrize("N,rows,cols,m0", [(3, 128, 128, 0), (20, 64, 64, 7), (64, 40, 32, 1000)])
def test_noise_segmented_bit_exact(dev_ops, N, rows, cols, m0):
    """Few substreams -> the segmented launch (chunks drawn by separate warps, chained in order):
    bit-identical to numpy's draws (C oracle) and to the one-warp-per-substream launch."""
    import os

    from oracle import noise as onoise
    from paper_2410_09663_b200.matvar import entropy_head

    assert dev_ops.lib.enks_noise_ws_bytes(N, 3, rows, cols) > 0  # takes the segmented path
    head = entropy_head(11, (2, 5))
    diag = dev_ops.to_device(np.linspace(0.5, 2.0, rows), dtype=torch.float64)
    base = torch.randn(rows, N * cols, device=dev_ops.device)

    def draw():
        outs = [dev_ops.zeros(rows, N * cols) for _ in range(3)]
        plus = dev_ops.zeros(rows, N * cols)
        dev_ops.noise_fill_multi(head, m0, N, cols, [
            dict(t=4, ch=0, rows=rows, diag=diag, out=outs[0], base=base, out_plus=plus),
            dict(t=4, ch=1, rows=rows, out=outs[1]), dict(t=4, ch=2, rows=rows, out=outs[2])])
        torch.cuda.synchronize()
        return outs, plus

    seg, seg_plus = draw()
    os.environ["ENKS_NOISE_SEG"] = "0"
    try:
        ref, ref_plus = draw()
    finally:
        del os.environ["ENKS_NOISE_SEG"]
    for a, b in zip(seg, ref):
        assert torch.equal(a, b)
    assert torch.equal(seg_plus, ref_plus)
    z = onoise.member_normals(11, (2, 5), 4, 1, m0 + N, (rows, cols), backend="c")[m0:]
    want = np.ascontiguousarray(z.transpose(1, 0, 2).reshape(rows, -1)).astype(np.float32)
    assert np.array_equal(seg[1].cpu().numpy(), want)


@pytest.mark.parametrize("rows,N", [(24, 300), (2, 150), (3, 149), (128, 20), (37, 4), (128, 64),
                                    (50, 9)])
def test_cnn_forward_tcgen05_several_images_per_cta(dev_ops, pm, rows, N):
    """128-pixel images with more images than SMs: each CTA streams several images through the
    same row pipeline (TMEM ring, A slots, tap ring continue across image boundaries); minimum
    image height 2 (both edge rows at once).  Fewer images than SMs: every image's rows are split
    into units with a two-row halo (7 uneven parts of 128 rows at N = 20, 2 parts at N = 64, ...),
    several units per CTA when parts x N > 148."""
    from oracle.models import cnn_step_torch
    from paper_2410_09663_b200.engine import Forecaster

    model = pm.dynamics.CNNDynamics(rows=rows, cols=128, widths=(2, 32, 32, 1), seed=5)
    model.state_rows = model.input_rows = rows
    rng = np.random.default_rng(N)
    x = rng.standard_normal((N, rows, 128))
    u = rng.standard_normal((N, rows, 128))
    ref = cnn_step_torch(x, u, model.weights, model.biases, model.alpha)
    last = dev_ops.to_device(np.concatenate([x, u], axis=1).transpose(1, 0, 2).reshape(2 * rows, -1))
    out = dev_ops.zeros(rows, N * 128)
    Forecaster(model, dev_ops, rows, rows)(dev_ops, last, out, rows, N)
    got = _cpu(out).reshape(rows, N, 128).transpose(1, 0, 2)
    np.testing.assert_allclose(got, ref, rtol=1e-5, atol=2e-6)


@pytest.mark.parametrize("rows,rows2,N,cols", [(384, 256, 1024, 128), (12, 8, 37, 8), (8, 0, 5, 4)])
def test_member_sum2_matches_two_passes(dev_ops, rows, rows2, N, cols):
    """One pass for the slice sums of src and the observation sums of src[:rows2] + src2 ==
    the two enks_member_sum passes (same values to fp64 rounding; amax exact)."""
    g = torch.Generator().manual_seed(rows + N)
    src = (torch.randn(rows, N * cols, generator=g) * 3 + 1).to(dev_ops.device)
    src2 = torch.randn(max(rows2, 1), N * cols, generator=g).to(dev_ops.device)
    acc1 = torch.zeros(rows, cols, dtype=torch.float64, device=dev_ops.device)
    amax1 = dev_ops.zeros(rows, cols)
    acc2 = torch.zeros(max(rows2, 1), cols, dtype=torch.float64, device=dev_ops.device)
    amax2 = dev_ops.zeros(max(rows2, 1), cols)
    dev_ops.member_sum2(src, rows2, src2, N, cols, acc1, amax1, acc2, amax2)
    r1 = torch.zeros_like(acc1)
    m1 = torch.zeros_like(amax1)
    dev_ops.member_sum(src, N, cols, None, r1, m1)
    torch.testing.assert_close(acc1, r1, rtol=1e-12, atol=1e-9)
    assert torch.equal(amax1, m1)
    if rows2:
        r2 = torch.zeros_like(acc2)
        m2 = torch.zeros_like(amax2)
        dev_ops.member_sum(src[:rows2], N, cols, None, r2, m2, src2=src2[:rows2])
        torch.testing.assert_close(acc2, r2, rtol=1e-12, atol=1e-9)
        assert torch.equal(amax2, m2)
