"""TEST-ONLY CPU restatement of the device operator interface (paper_2410_09663_b200/ops.py).

Lets the engine's orchestration (the append-only basis algebra, member
sharding, collectives) run on CPU with the gloo backend, where no GPU
exists.  Each method restates the contract of the matching C-ABI entry
point (include/enks_b200.h) in fp64 torch; noise comes from the C oracle.
Never imported by the product package.
"""
from __future__ import annotations

import numpy as np
import torch

from oracle import noise as onoise


class CpuOps:
    dtype = torch.float64

    def __init__(self):
        self.device = torch.device("cpu")
        self.launches = 0

    # fp16-pair basis buffers are kept in fp64 here (h = x, l = 0, scale 1): the
    # orchestration of the pair path is exercised exactly, without fp16 rounding
    def empty(self, *shape, dtype=None):
        return torch.empty(shape, dtype=self.dtype if dtype in (None, torch.float16) else dtype)

    def zeros(self, *shape, dtype=None):
        return torch.zeros(shape, dtype=self.dtype if dtype in (None, torch.float16) else dtype)

    def f16pair_split(self, src, h, l, inv_scale):
        h.copy_(src)
        l.zero_()
        inv_scale.fill_(1.0)

    def f16pair_recon(self, h, l, inv_scale, out):
        out.copy_((h + l) * inv_scale[:, None])

    def gemm_f16pair(self, Ah, Al, inv_sa, Bh, Bl, inv_sb, C, *, alpha=1.0, tag=None):
        a = (Ah + Al) * inv_sa[:, None]
        b = (Bh + Bl) * inv_sb[:, None]
        C.copy_(alpha * (a @ b.t()))

    def f16pair_transpose(self, h, l, inv_src, oh, ol, inv_out):
        oh.copy_(((h + l) * inv_src[:, None]).t())
        ol.zero_()
        inv_out.fill_(1.0)

    def gemm_f16pair_ex(self, Ah, Al, inv_sa, Bh, Bl, inv_sb, C, *, alpha=1.0, beta=0.0, C0=None,
                        bias=None, bias_cols=0, tag=None):
        a = (Ah + Al) * inv_sa[:, None]
        b = (Bh + Bl) * inv_sb[:, None]
        out = alpha * (a @ b.t())
        if C0 is not None:
            out = out + beta * C0
        if bias is not None:
            out = out + bias[:, torch.arange(out.shape[1]) % bias_cols]
        C.copy_(out)

    def member_center_f16pair(self, src, n_members, cols, z0, acc, amax, n_total, mean, h, l,
                              inv_scale, f32=None, rows_f32=0, skip=(0, 0)):
        anom = torch.empty(src.shape, dtype=self.dtype)
        self.member_center(src, n_members, cols, z0, acc, n_total, mean=mean, anom=anom)
        if f32 is not None and rows_f32:
            f32[:rows_f32].copy_(anom[:rows_f32])
        if skip[1] > skip[0]:
            anom = torch.cat([anom[:skip[0]], anom[skip[1]:]])
        h.copy_(anom)
        l.zero_()
        inv_scale.fill_(1.0)

    def member_center_f16pair_t(self, src, src2, n_members, cols, z0, acc, amax, n_total, mean, h,
                                l, inv_scale, th, tl, t_inv):
        anom = torch.empty(src.shape, dtype=self.dtype)
        self.member_center(src + src2, n_members, cols, z0, acc, n_total, mean=mean, anom=anom)
        h.copy_(anom)
        l.zero_()
        inv_scale.fill_(1.0)
        th.copy_(anom.t())
        tl.zero_()
        t_inv.fill_(1.0)

    def uchain_apply(self, delta, mean, gcol, gtt, n_slices, n, l, m, p):
        ds, d = n + l, n + 2 * l
        dc = delta[:n_slices * ds].reshape(n_slices, ds, m)
        mv = mean[:n_slices * d].view(n_slices, d, m)
        mv[:, :n] += dc[:, :n]
        mv[:, n + l:] += dc[:, n:]
        mv[:, n:n + l] += torch.cumsum(dc[:, n:], dim=0)
        gc = gcol[:n_slices * ds].reshape(n_slices, ds, p)
        gtt[:n].copy_(gc[-1, :n])
        gtt[n:n + l].copy_(gc[:, n:].sum(dim=0))

    def to_device(self, arr, dtype=None):
        arr = np.require(arr, requirements=["C", "W"])
        return torch.as_tensor(arr, dtype=dtype or self.dtype).clone()

    def copy_from_host(self, dst, arr):
        dst.copy_(torch.from_numpy(np.ascontiguousarray(arr)).to(dst.dtype))

    def to_host(self, t):
        return t.double().numpy()

    def read_scalar(self, t):
        return t.item()

    def noise_fill(self, head, t, ch, member0, n_members, rows, cols, diag=None, out=None,
                   base=None, out_plus=None):
        out_z = np.empty((n_members, rows * cols))
        for k in range(n_members):
            ent = list(head) + [member0 + k, t, ch]
            key = np.zeros(2, dtype=np.uint64)
            import ctypes

            arr = np.asarray(ent, dtype=np.uint32)
            onoise._lib().npyo_seedseq_key(arr.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                           len(arr),
                                           key.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
            onoise._lib().npyo_standard_normal(key.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                               rows * cols,
                                               out_z[k].ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        z = out_z.reshape(n_members, rows, cols)
        if diag is not None:
            z = z * diag.numpy()[None, :, None]
        blk = torch.from_numpy(np.ascontiguousarray(z.transpose(1, 0, 2).reshape(rows, -1)))
        if out is not None:
            out.copy_(blk)
        if out_plus is not None:
            out_plus.copy_(base + blk)

    def noise_fill_multi(self, head, member0, n_members, cols, jobs):
        for j in jobs:
            self.noise_fill(head, j["t"], j["ch"], member0, n_members, j["rows"], cols,
                            diag=j.get("diag"), out=j.get("out"), base=j.get("base"),
                            out_plus=j.get("out_plus"))

    def add(self, a, b, out):
        out.copy_(a + b)

    def member_sum(self, src, n_members, cols, z0, acc, amax=None, src2=None):
        if src2 is not None:
            src = src + src2
        s = src.reshape(src.shape[0], n_members, cols)
        shift = s[:, 0, :] if z0 is None else z0
        acc.copy_((s - shift[:, None, :]).sum(dim=1))
        if amax is not None:
            amax.copy_((s - shift[:, None, :]).abs().amax(dim=1))

    def member_sum_rebase(self, src, cols, acc, coef, src2=None):
        s = src[:acc.shape[0], :cols] + (src2[:acc.shape[0], :cols] if src2 is not None else 0)
        acc.add_(coef * s)

    def member_center(self, src, n_members, cols, z0, acc, n_total, mean=None, anom=None):
        s = src.reshape(src.shape[0], n_members, cols)
        shift = (s[:, 0, :] if z0 is None else z0).clone()
        mu = acc / n_total
        if mean is not None:
            mean.copy_(shift + mu)
        if anom is not None:
            anom.copy_(((s - shift[:, None, :]) - mu[:, None, :]).reshape(anom.shape))

    def gemm(self, A, B, C, *, trans_a=False, trans_b=False, alpha=1.0, beta=0.0, C0=None,
             bias=None, bias_cols=1, tri=(0, 0), split=None, engine=0, tag=None):
        a = A.t() if trans_a else A
        b = B.t() if trans_b else B
        if a.shape[1] == 0:
            prod = torch.zeros(C.shape, dtype=C.dtype)
        else:
            prod = alpha * (a @ b)
        if C0 is not None:
            prod = prod + beta * C0
        if bias is not None:
            reps = C.shape[1] // bias_cols
            prod = prod + bias[:, :bias_cols].repeat(1, reps)
        C.copy_(prod)

    def spd_inverse(self, S, scale, inv, status, jitter):
        sy = scale * 0.5 * (S + S.t())
        p = sy.shape[0]
        try:
            L = torch.linalg.cholesky(sy)
        except RuntimeError:
            j = 1e-9 * float(torch.trace(sy)) / p + 1e-30
            jitter += 1
            L = torch.linalg.cholesky(sy + j * torch.eye(p, dtype=sy.dtype))
        inv.copy_(torch.cholesky_inverse(L))

    def spd_max_p(self):
        return 1 << 30

    def cnn_forward(self, cnn, x, u, out, n_members):
        from oracle.models import cnn_step

        n, m = x.shape[0], cnn.cols
        xs = x.numpy().reshape(n, n_members, m).transpose(1, 0, 2)
        us = u.numpy().reshape(n, n_members, m).transpose(1, 0, 2)
        w = [np.asarray(v) for v in cnn.model.weights]
        b = [np.asarray(v) for v in cnn.model.biases]
        y = cnn_step(xs, us, w, b, cnn.alpha)
        out.copy_(torch.from_numpy(np.ascontiguousarray(y.transpose(1, 0, 2).reshape(n, -1))))

    def burgers_forward(self, bur, x, u, out, n_members):
        from oracle.models import burgers_step

        g = bur.grid_n
        xs = x.numpy().reshape(2 * g, n_members, g).transpose(1, 0, 2)
        us = u.numpy().reshape(u.shape[0], n_members, g).transpose(1, 0, 2)
        mode = "pointwise" if u.shape[0] == 2 * g else "boundary"
        y, vmax = burgers_step(xs, us, g, bur.nu, bur.dt, mode, bur.substeps)
        bur.vmax[0] = max(float(bur.vmax[0]), vmax)
        out.copy_(torch.from_numpy(np.ascontiguousarray(y.transpose(1, 0, 2).reshape(2 * g, -1))))

    def barrier_row(self, bar, S, n, l, m, n_members, eps, out):
        import math

        d = n + 2 * l
        Sm = S.numpy().reshape(d, n_members, m)
        for i in range(n_members):
            blk = Sm[bar.r0:bar.r1, i, :]
            if bar.kind == 0:
                g = float(np.sum(bar.coef.numpy()[bar.r0:bar.r1] * blk)) + bar.c0
            else:
                g = float(np.max(np.abs(blk))) + bar.c0
            z = bar.beta * g
            clean = z / bar.alpha if z > 30.0 else math.log1p(math.exp(z)) / bar.alpha
            out[0, i * m:(i + 1) * m] = clean + bar.sqrt_var * float(eps[0, i])

    def quad_form(self, E, X, out, scale=1.0, accumulate=False):
        v = scale * float((E.double() * X.double()).sum())
        out[0] = (float(out[0]) if accumulate else 0.0) + v

    def sub(self, a, b, out):
        out.copy_(a - b)
