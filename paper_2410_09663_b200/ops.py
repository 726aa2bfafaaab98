"""Device operator set: thin tensor-view wrappers over the C-ABI (include/enks_b200.h).

The smoother engine (``engine.py``) is written against this small operator
interface.  ``DeviceOps`` is the only implementation in the product; every
method is one or two stream-ordered launches of an sm_100a kernel through
ctypes.  (tests/cpu_ops.py holds a CPU restatement of the same interface
used ONLY to exercise the multi-rank orchestration with the gloo backend.)

Tensor arguments are 2-D views with unit column stride; the row stride is
passed as the leading dimension.
"""
from __future__ import annotations

import contextlib
import ctypes

import numpy as np
import torch

from . import _lib

NUM_SMS = 148


def _ld(t: torch.Tensor) -> int:
    if t.dim() != 2 or (t.shape[1] > 1 and t.stride(1) != 1):
        raise ValueError(f"expected a 2-D row-major view, got shape {tuple(t.shape)} "
                         f"strides {t.stride()}")
    return t.stride(0) if t.shape[0] > 1 else max(t.shape[1], t.stride(0))


def _p(t):
    return None if t is None else t.data_ptr()


class DeviceHead:
    """Noise entropy words kept in device memory (int32 tensor, first n used): a captured CUDA
    graph reads them at replay, so one capture serves every NoiseStreams.child(k)."""

    def __init__(self, words, n: int):
        self.words, self.n = words, int(n)

    def set(self, host_words) -> None:
        w = [int(x) for x in host_words]
        if len(w) != self.n:
            raise ValueError(f"head has {len(w)} words, the capture used {self.n}")
        self.words[:self.n].copy_(torch.tensor(np.array(w, dtype=np.uint32).view(np.int32)))


def choose_split(M: int, N: int, K: int, bm: int = 128, bn: int = 128, min_k: int = 2048) -> int:
    """Split-K factor so that a tall-skinny contraction fills the 148 SMs (>= 2 waves)."""
    tiles = -(-M // bm) * -(-N // bn)
    if tiles >= 2 * NUM_SMS:
        return 1
    split = -(-2 * NUM_SMS // tiles)
    return int(max(1, min(split, K // min_k, 128)))


class DeviceOps:
    """sm_100a kernels behind the C-ABI.  No CPU fallback: construction fails loudly."""

    dtype = torch.float32

    def __init__(self, device: torch.device | int | None = None):
        self.lib = _lib.load_library(check_device=True)
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        self._ws = None
        self._ws_sum = None
        # workspaces replaced by larger ones are retained (never freed): a captured CUDA graph
        # (enks.HorizonGraph) may still hold their addresses
        self._retired = []
        self.launches = 0  # kernel launches issued through the C-ABI (bench's gpu_launches)
        self.h2d_bytes = 0  # host<->device bytes moved by the product (bench's e2e accounting)
        self.d2h_bytes = 0
        self.profile = None  # list -> (tag, start_event, end_event, algorithmic_flops) per tagged op

    # -- memory -----------------------------------------------------------
    def empty(self, *shape, dtype=None):
        return torch.empty(shape, dtype=dtype or self.dtype, device=self.device)

    def zeros(self, *shape, dtype=None):
        return torch.zeros(shape, dtype=dtype or self.dtype, device=self.device)

    def to_device(self, arr, dtype=None):
        arr = np.require(arr, requirements=["C", "W"])  # (copies read-only broadcast views)
        t = torch.as_tensor(arr, dtype=dtype or self.dtype)
        self.h2d_bytes += t.numel() * t.element_size()
        return t.to(self.device)

    def copy_from_host(self, dst, arr) -> None:
        """dst (device) <- host array, converted to dst's dtype on the host first."""
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(dst.dtype)
        self.h2d_bytes += t.numel() * t.element_size()
        dst.copy_(t)

    def to_host(self, t) -> np.ndarray:
        """Device tensor -> fp64 NumPy.  Results up to 64 MB (mean trajectories, P / G blocks) are
        widened on the device and copied once into pinned memory (torch's cached pinned pool; the
        array keeps its buffer alive); larger ones (tracked covariances) are copied in their own
        dtype and widened on the host, without a pinned / fp64 device copy of their size."""
        if t.is_cuda and t.numel() * 8 <= (64 << 20):
            h = torch.empty(t.shape, dtype=torch.float64, pin_memory=True)
            h.copy_(t.double())
            self.d2h_bytes += h.numel() * h.element_size()
            return h.numpy()
        self.d2h_bytes += t.numel() * t.element_size()
        return t.cpu().double().numpy()

    def read_scalar(self, t):
        self.d2h_bytes += t.element_size()
        return t.item()

    def _workspace(self, nbytes: int) -> int:
        if nbytes <= 0:
            return 0
        if self._ws is None or self._ws.numel() < nbytes:
            self._retire(self._ws)
            self._ws = torch.empty(int(nbytes * 1.25) + 256, dtype=torch.uint8, device=self.device)
        return self._ws.data_ptr()

    def _retire(self, buf) -> None:
        if buf is not None:
            self._retired.append(buf)

    def _workspace_sum(self, nbytes: int) -> int:
        if self._ws_sum is None or self._ws_sum.numel() < nbytes:
            self._retire(self._ws_sum)
            self._ws_sum = torch.empty(int(nbytes * 1.25) + 256, dtype=torch.uint8,
                                       device=self.device)
        return self._ws_sum.data_ptr()

    @staticmethod
    def _stream() -> int:
        return torch.cuda.current_stream().cuda_stream

    @contextlib.contextmanager
    def _prof(self, tag, work):
        """CUDA-event bracket of one op when profiling (bench): (tag, ev0, ev1, work)."""
        if self.profile is None:
            yield
            return
        ev0 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        yield
        ev1 = torch.cuda.Event(enable_timing=True)
        ev1.record()
        self.profile.append((tag, ev0, ev1, float(work)))

    # -- kernels ----------------------------------------------------------
    def noise_fill(self, head, t, ch, member0, n_members, rows, cols, diag=None, out=None,
                   base=None, out_plus=None):
        if isinstance(head, DeviceHead):
            self.noise_fill_multi(head, member0, n_members, cols, [dict(
                t=t, ch=ch, rows=rows, diag=diag, out=out, base=base, out_plus=out_plus)])
            return
        words = (ctypes.c_uint32 * len(head))(*[int(w) for w in head])
        self.launches += 1
        with self._prof("noise", rows * cols * n_members):  # work = normals drawn
            self._noise_fill(words, head, t, ch, member0, n_members, rows, cols, diag, out, base,
                             out_plus)

    def _noise_fill(self, words, head, t, ch, member0, n_members, rows, cols, diag, out, base,
                    out_plus):
        _lib.call("enks_noise_fill", words, len(head), int(t), int(ch), int(member0),
                  int(n_members), int(rows), int(cols), _p(diag), _p(out),
                  _ld(out) if out is not None else 0, _p(base),
                  _ld(base) if base is not None else 0, _p(out_plus),
                  _ld(out_plus) if out_plus is not None else 0, self._stream())

    def noise_fill_multi(self, head, member0, n_members, cols, jobs):
        """jobs: list of dicts (t, ch, rows, diag, out, base, out_plus); one launch."""
        n = len(jobs)
        words = None if isinstance(head, DeviceHead) else \
            (ctypes.c_uint32 * len(head))(*[int(w) for w in head])
        u32 = ctypes.c_uint32 * n
        vp = ctypes.c_void_p * n
        i64 = ctypes.c_int64 * n
        get = lambda k: [j.get(k) for j in jobs]  # noqa: E731
        self.launches += 1
        with self._prof("noise", sum(j["rows"] * cols * n_members for j in jobs)):  # normals
            self._noise_multi(words, head, member0, n_members, cols, n, u32, vp, i64, get, jobs)

    def _noise_multi(self, words, head, member0, n_members, cols, n, u32, vp, i64, get, jobs):
        if isinstance(head, DeviceHead):
            fn, words, n_head = "enks_noise_fill_multi_dev", _p(head.words), head.n
        else:
            fn, n_head = "enks_noise_fill_multi", len(head)
        # segmented launch workspace (few substreams: chunks drawn by separate warps)
        wsb = int(self.lib.enks_noise_ws_bytes(int(n_members), n, max(int(j["rows"]) for j in jobs),
                                               int(cols)))
        ws = None
        if wsb:
            if getattr(self, "_noise_ws", None) is None or self._noise_ws.numel() < wsb:
                self._retire(getattr(self, "_noise_ws", None))
                self._noise_ws = torch.empty(wsb, dtype=torch.uint8, device=self.device)
            ws = self._noise_ws
        _lib.call(fn, words, n_head, int(member0), int(n_members), int(cols),
                  n, u32(*[int(j["t"]) for j in jobs]), u32(*[int(j["ch"]) for j in jobs]),
                  (ctypes.c_int * n)(*[int(j["rows"]) for j in jobs]),
                  vp(*[_p(v) for v in get("diag")]), vp(*[_p(v) for v in get("out")]),
                  i64(*[_ld(v) if v is not None else 0 for v in get("out")]),
                  vp(*[_p(v) for v in get("base")]),
                  i64(*[_ld(v) if v is not None else 0 for v in get("base")]),
                  vp(*[_p(v) for v in get("out_plus")]),
                  i64(*[_ld(v) if v is not None else 0 for v in get("out_plus")]),
                  _p(ws), int(wsb), self._stream())

    def member_sum(self, src, n_members, cols, z0, acc, amax=None, src2=None):
        """Member sums of src (+ src2, formed on the fly) relative to z0 (or member 0)."""
        rows = src.shape[0]
        nbytes = self.lib.enks_member_sum_ws_bytes(rows, n_members, cols)
        ws = self._workspace_sum(nbytes)
        self.launches += 2
        nsrc = 1 if src2 is None else 2
        with self._prof("stats", 4 * nsrc * rows * n_members * cols):
            _lib.call("enks_member_sum", _p(src), _ld(src), _p(src2),
                      _ld(src2) if src2 is not None else 0, rows, int(n_members), int(cols),
                      _p(z0), _p(acc), _p(amax), ws, self._stream())

    def member_sum2(self, src, rows2, src2, n_members, cols, acc, amax, acc2, amax2):
        """Slice sums of src and observation sums of src[:rows2] + src2 in one pass."""
        rows = src.shape[0]
        nbytes = self.lib.enks_member_sum2_ws_bytes(rows, int(rows2), int(n_members), int(cols))
        ws = self._workspace_sum(nbytes)
        self.launches += 3
        with self._prof("stats", 4 * (rows + rows2) * n_members * cols):
            _lib.call("enks_member_sum2", _p(src), _ld(src), rows, _p(src2), _ld(src2), int(rows2),
                      int(n_members), int(cols), _p(acc), _p(amax), _p(acc2), _p(amax2), ws,
                      self._stream())

    def member_sum_rebase(self, src, cols, acc, coef, src2=None):
        """acc += coef * (local member 0 of src (+ src2)): shifted <-> absolute member sums."""
        self.launches += 1
        _lib.call("enks_member_sum_rebase", _p(src), _ld(src), _p(src2),
                  _ld(src2) if src2 is not None else 0, int(acc.shape[0]), int(cols), _p(acc),
                  float(coef), self._stream())

    def member_center_f16pair_t(self, src, src2, n_members, cols, z0, acc, amax, n_total, mean, h,
                                l, inv_scale, th, tl, t_inv):
        """Centring of src + src2 into the pair basis rows and transposed pair planes."""
        rows = src.shape[0]
        if getattr(self, "_scale_ws", None) is None or self._scale_ws.numel() < rows:
            self._retire(getattr(self, "_scale_ws", None))
            self._scale_ws = torch.empty(max(rows, 4096), dtype=torch.float32, device=self.device)
        self.launches += 2
        K = n_members * cols
        with self._prof("stats", 8 * rows * K + 8 * rows * K):
            _lib.call("enks_member_center_f16pair_t", _p(src), _ld(src), _p(src2), _ld(src2), rows,
                      int(n_members), int(cols), _p(z0), _p(acc), _p(amax), int(n_total), _p(mean),
                      _p(h), _p(l), _ld(h), _p(inv_scale), _p(self._scale_ws), _p(th), _p(tl),
                      _ld(th) if th is not None else 0, _p(t_inv), self._stream())

    def member_center_f16pair(self, src, n_members, cols, z0, acc, amax, n_total, mean, h, l,
                              inv_scale, f32=None, rows_f32=0, skip=(0, 0)):
        rows = src.shape[0]
        if getattr(self, "_scale_ws", None) is None or self._scale_ws.numel() < rows:
            self._retire(getattr(self, "_scale_ws", None))
            self._scale_ws = torch.empty(max(rows, 4096), dtype=torch.float32, device=self.device)
        self.launches += 2
        K = n_members * cols
        with self._prof("stats", 8 * rows * K + 4 * rows_f32 * K):
            _lib.call("enks_member_center_f16pair", _p(src), _ld(src), rows, int(n_members),
                      int(cols), _p(z0), _p(acc), _p(amax), int(n_total), _p(mean), _p(h), _p(l),
                      _ld(h), _p(inv_scale), _p(self._scale_ws), _p(f32),
                      _ld(f32) if f32 is not None else 0, int(rows_f32), int(skip[0]),
                      int(skip[1]), self._stream())

    def uchain_apply(self, delta, mean, gcol, gtt, n_slices, n, l, m, p):
        """Derived-U chain (stats.cu): mean += delta with prefix-summed U rows; gtt = newest
        slice's [X; U] gain rows from the compact gain column."""
        self.launches += 2
        _lib.call("enks_uchain_apply", _p(delta), _ld(delta), _p(mean), _ld(mean), _p(gcol),
                  _ld(gcol), _p(gtt), _ld(gtt), int(n_slices), int(n), int(l), int(m), int(p),
                  self._stream())

    def member_center(self, src, n_members, cols, z0, acc, n_total, mean=None, anom=None):
        rows = src.shape[0]
        self.launches += 1
        _lib.call("enks_member_center", _p(src), _ld(src), rows, int(n_members), int(cols),
                  _p(z0), _p(acc), int(n_total), _p(mean), _p(anom),
                  _ld(anom) if anom is not None else 0, self._stream())

    def gemm(self, A, B, C, *, trans_a=False, trans_b=False, alpha=1.0, beta=0.0, C0=None,
             bias=None, bias_cols=1, tri=(0, 0), split=None, engine=0, tag=None):
        M, N = C.shape
        K = A.shape[0] if trans_a else A.shape[1]
        if (B.shape[1] if trans_b else B.shape[0]) != K:
            raise ValueError("gemm: inner dimensions disagree")
        if M == 0 or N == 0:
            return
        if split is None:
            split = choose_split(M, N, K)
        ws = self._workspace(self.lib.enks_gemm_ws_bytes(M, N, split)) if split > 1 else None
        self.launches += 2 if split > 1 else 1
        prof = self.profile is not None and tag is not None
        if prof:
            ev0 = torch.cuda.Event(enable_timing=True)
            ev0.record()
        _lib.call("enks_gemm", int(trans_a), int(trans_b), M, N, K, float(alpha),
                  _p(A) if K else None, _ld(A) if K else 0, _p(B) if K else None,
                  _ld(B) if K else 0, float(beta), _p(C0), _ld(C0) if C0 is not None else 0,
                  _p(bias), _ld(bias) if bias is not None else 0, int(bias_cols), _p(C), _ld(C),
                  int(tri[0]), int(tri[1]), int(split), ws, int(engine), self._stream())
        if prof:
            ev1 = torch.cuda.Event(enable_timing=True)
            ev1.record()
            self.profile.append((tag, ev0, ev1, 2.0 * M * N * K))

    def tc_applicable(self, A, Bh) -> bool:
        """tcgen05 3xTF32 path: N <= 256, K >= 128, 16-B aligned rows."""
        K = A.shape[1]
        return (Bh.shape[0] <= 256 and K >= 128 and _ld(A) % 4 == 0 and _ld(Bh) % 4 == 0
                and A.data_ptr() % 16 == 0 and Bh.data_ptr() % 16 == 0)

    def tf32_split(self, src, hi, lo, transpose=False):
        """hi = rna_tf32(src), lo = src - hi (B operand of the 3xTF32 GEMMs); transpose=True
        writes the (cols x rows) planes, i.e. the K-major form of a K x N operand."""
        self.launches += 1
        _lib.call("enks_tf32_split", _p(src), _ld(src), src.shape[0], src.shape[1], _p(hi), _p(lo),
                  int(transpose), self._stream())

    def gemm_nt_tc(self, A, Bh, Bl, C, *, alpha=1.0, split=0, tag=None):
        """C = alpha * A (Bh + Bl)^T on tcgen05 (3xTF32), deterministic split-K."""
        M, K = A.shape
        N = Bh.shape[0]
        if M == 0 or N == 0:
            return
        ws = self._workspace(self.lib.enks_tc_gemm_ws_bytes(M, N, K, int(split)))
        self.launches += 2
        prof = self.profile is not None and tag is not None
        if prof:
            ev0 = torch.cuda.Event(enable_timing=True)
            ev0.record()
        _lib.call("enks_gemm_nt_tc", M, N, K, float(alpha), _p(A), _ld(A), _p(Bh), _p(Bl), _ld(Bh),
                  _p(C), _ld(C), int(split), ws, self._stream())
        if prof:
            ev1 = torch.cuda.Event(enable_timing=True)
            ev1.record()
            self.profile.append((tag, ev0, ev1, 2.0 * M * N * K))

    def gemm_tc(self, A, Bh, Bl, C, *, alpha=1.0, beta=0.0, C0=None, bias=None, bias_cols=1,
                tri=(0, 0), split=0, tag=None):
        """C = alpha * A (Bh + Bl)^T + beta * C0 + bias on tcgen05 (3xTF32).

        Bh/Bl are the K-major (N x K) planes of B (see tf32_split(transpose=True))."""
        M, K = A.shape
        N = Bh.shape[0]
        if M == 0 or N == 0:
            return
        if split == 0:
            tiles = -(-M // 128) * -(-N // 256)
            split = 1 if tiles >= NUM_SMS or K < 1024 else int(min(-(-NUM_SMS // tiles), K // 512))
        ws = self._workspace(int(split) * M * N * 4) if split > 1 else None
        self.launches += 2 if split > 1 else 1
        prof = self.profile is not None and tag is not None
        if prof:
            ev0 = torch.cuda.Event(enable_timing=True)
            ev0.record()
        _lib.call("enks_gemm_tc", M, N, K, float(alpha), _p(A), _ld(A), _p(Bh), _p(Bl), _ld(Bh), 0,
                  float(beta), _p(C0), _ld(C0) if C0 is not None else 0, _p(bias),
                  _ld(bias) if bias is not None else 0, int(bias_cols), _p(C), _ld(C),
                  int(tri[0]), int(tri[1]), int(split), ws, self._stream())
        if prof:
            ev1 = torch.cuda.Event(enable_timing=True)
            ev1.record()
            self.profile.append((tag, ev0, ev1, 2.0 * M * N * K))

    # -- fp16-pair basis (gemm_f16p.cu) -------------------------------------
    def f16pair_split(self, src, h, l, inv_scale):
        """Per-row power-of-two scaled (hi, lo) fp16 planes of src (rows x K)."""
        self.launches += 1
        _lib.call("enks_f16pair_split", _p(src), _ld(src), src.shape[0], src.shape[1], _p(h), _p(l),
                  _ld(h), _p(inv_scale), self._stream())

    def f16pair_split_cs(self, src, col_scale, h, l, inv_scale):
        """f16pair_split of src * col_scale (per column) -- e.g. G_tt with Yc_tau's row scale."""
        self.launches += 1
        _lib.call("enks_f16pair_split_cs", _p(src), _ld(src), src.shape[0], src.shape[1],
                  _p(col_scale), _p(h), _p(l), _ld(h), _p(inv_scale), self._stream())

    def ones(self, n: int):
        """A cached device vector of n ones (fp32)."""
        o = getattr(self, "_ones", None)
        if o is None or o.numel() < n:
            self._retire(o)
            self._ones = o = torch.ones(int(n), device=self.device)
        return o[:n]

    def f16pair_recon(self, h, l, inv_scale, out):
        self.launches += 1
        _lib.call("enks_f16pair_recon", _p(h), _p(l), _ld(h), _p(inv_scale), out.shape[0],
                  out.shape[1], _p(out), _ld(out), self._stream())

    def set_sm_reserve(self, sms: int) -> None:
        """SMs left free in the next cross-moment grids (enks_set_sm_reserve)."""
        _lib.call("enks_set_sm_reserve", int(sms))

    def gemm_f16pair(self, Ah, Al, inv_sa, Bh, Bl, inv_sb, C, *, alpha=1.0, tag=None):
        """C = alpha * diag(inv_sa) (Ah + Al)(Bh + Bl)^T diag(inv_sb), tcgen05 kind::f16."""
        M, K = Ah.shape
        N = Bh.shape[0]
        if M == 0:
            return
        nbytes = self.lib.enks_gemm_f16pair_ws_bytes(M, N, K)
        ws = self._workspace(nbytes) if nbytes > 0 else None
        self.launches += 2 if nbytes > 0 else 1
        prof = self.profile is not None and tag is not None
        if prof:
            ev0 = torch.cuda.Event(enable_timing=True)
            ev0.record()
        _lib.call("enks_gemm_f16pair", M, N, K, float(alpha), _p(Ah), _p(Al), _ld(Ah), _p(inv_sa),
                  _p(Bh), _p(Bl), _ld(Bh), _p(inv_sb), _p(C), _ld(C), ws, self._stream())
        if prof:
            ev1 = torch.cuda.Event(enable_timing=True)
            ev1.record()
            self.profile.append((tag, ev0, ev1, 2.0 * M * N * K))

    def f16pair_transpose(self, h, l, inv_src, oh, ol, inv_out):
        """(h + l) * inv_src (rows x K fp16 pairs, rows <= 256) -> transposed planes (K x rows)."""
        self.launches += 1
        _lib.call("enks_f16pair_transpose", _p(h), _p(l), _ld(h), _p(inv_src), h.shape[0],
                  h.shape[1], _p(oh), _p(ol), _ld(oh), _p(inv_out), self._stream())

    def gemm_f16pair_ex(self, Ah, Al, inv_sa, Bh, Bl, inv_sb, C, *, alpha=1.0, beta=0.0, C0=None,
                        bias=None, bias_cols=0, tag=None):
        """C = alpha A B^T (fp16-pair planes, any N) + beta C0 + bias[:, c % bias_cols]."""
        M, K = Ah.shape
        N = Bh.shape[0]
        if M == 0:
            return
        self.launches += 1
        with self._prof(tag, 2.0 * M * N * K) if tag else contextlib.nullcontext():
            _lib.call("enks_gemm_f16pair_ex", M, N, K, float(alpha), _p(Ah), _p(Al), _ld(Ah),
                      _p(inv_sa), _p(Bh), _p(Bl), _ld(Bh), _p(inv_sb), float(beta), _p(C0),
                      _ld(C0) if C0 is not None else 0, _p(bias),
                      _ld(bias) if bias is not None else 0, int(bias_cols), _p(C), _ld(C),
                      self._stream())

    def gemm_f16pair_ex_mn(self, Ah, Al, inv_sa, Bh, Bl, C, *, alpha=1.0, beta=0.0, C0=None,
                           bias=None, bias_cols=0, tag=None):
        """C = alpha A B + beta C0 + bias[:, c % bias_cols] with B given K x N (MN-major fp16
        pairs, no per-row scale of B: fold it into A); N > 128."""
        M, K = Ah.shape
        N = Bh.shape[1]
        if M == 0:
            return
        self.launches += 1
        with self._prof(tag, 2.0 * M * N * K) if tag else contextlib.nullcontext():
            _lib.call("enks_gemm_f16pair_ex_mn", M, N, K, float(alpha), _p(Ah), _p(Al), _ld(Ah),
                      _p(inv_sa), _p(Bh), _p(Bl), _ld(Bh), _p(self.ones(N)), float(beta), _p(C0),
                      _ld(C0) if C0 is not None else 0, _p(bias),
                      _ld(bias) if bias is not None else 0, int(bias_cols), _p(C), _ld(C),
                      self._stream())

    def gemm_nt_f16pair(self, a, b, out, *, alpha=1.0, tag=None):
        """out (M x N) = alpha a b^T for fp32 a (M x K), b (N x K) on tcgen05: both operands
        split into fp16-pair planes once, N covered in 256-column launches (any N)."""
        M, K = a.shape
        N = b.shape[0]
        f16 = torch.float16
        ah, al, sa = self.empty(M, K, dtype=f16), self.empty(M, K, dtype=f16), self.empty(M)
        self.f16pair_split(a, ah, al, sa)
        if b is a:
            bh, bl, sb = ah, al, sa
        else:
            bh, bl, sb = self.empty(N, K, dtype=f16), self.empty(N, K, dtype=f16), self.empty(N)
            self.f16pair_split(b, bh, bl, sb)
        for j0 in range(0, N, 256):
            j1 = min(N, j0 + 256)
            self.gemm_f16pair(ah, al, sa, bh[j0:j1], bl[j0:j1], sb[j0:j1], out[:, j0:j1],
                              alpha=alpha, tag=tag)

    def spd_inverse(self, S, scale, inv, status, jitter):
        p = S.shape[0]
        nf = (int(self.lib.enks_spd_ws_bytes(p)) + 3) // 4
        if getattr(self, "_spd_ws", None) is None or self._spd_ws.numel() < nf:
            self._retire(getattr(self, "_spd_ws", None))
            self._spd_ws = torch.empty(nf, dtype=torch.float32, device=self.device)
        self.launches += 2
        with self._prof("gain_solve", p ** 3 * (1.0 / 3 + 1.0 / 3 + 1.0)):
            self._spd(S, p, scale, inv, status, jitter)

    def _spd(self, S, p, scale, inv, status, jitter):
        _lib.call("enks_spd_inverse", _p(S), _ld(S), p, float(scale), _p(inv), _p(self._spd_ws),
                  _p(status), _p(jitter), self._stream())

    def spd_max_p(self) -> int:
        return int(self.lib.enks_spd_max_p())

    def cnn_forward(self, cnn, x, u, out, n_members):
        widths = (ctypes.c_int * len(cnn.widths))(*cnn.widths)
        self.launches += 1
        flops = n_members * x.shape[0] * cnn.cols * sum(
            18 * a * b for a, b in zip(cnn.widths[:-1], cnn.widths[1:]))
        wsb = int(self.lib.enks_cnn_ws_bytes(cnn.n_layers, widths, int(x.shape[0]), int(cnn.cols),
                                             int(n_members)))
        ws = None
        if wsb:
            if getattr(self, "_cnn_ws", None) is None or self._cnn_ws.numel() < wsb:
                self._retire(getattr(self, "_cnn_ws", None))
                self._cnn_ws = torch.empty(wsb, dtype=torch.uint8, device=self.device)
            ws = self._cnn_ws
            self.launches += 2 + cnn.n_layers
        with self._prof("forecast", flops):
            _lib.call("enks_cnn_forward_ws", cnn.n_layers, widths, _p(cnn.w_dev), _p(cnn.b_dev),
                      float(cnn.alpha), _p(x), _ld(x), _p(u), _ld(u), _p(out), _ld(out),
                      int(x.shape[0]), int(cnn.cols), int(n_members), _p(ws), int(wsb),
                      self._stream())

    def cnn_noise_fusable(self, cnn, rows) -> bool:
        """True when the fused 2-32-32-1 forecast can also draw the step's noise (cnn_tc.cu)."""
        widths = (ctypes.c_int * len(cnn.widths))(*cnn.widths)
        return bool(self.lib.enks_cnn_noise_fusable(cnn.n_layers, widths, int(rows), int(cnn.cols)))

    def cnn_forward_noise(self, cnn, x, u, out, n_members, head, member0, jobs):
        """Forecast out = f(x, u) with the noise jobs (as noise_fill_multi) drawn by the same
        launch's otherwise idle warps: one kernel instead of two that share SMs by time."""
        widths = (ctypes.c_int * len(cnn.widths))(*cnn.widths)
        n = len(jobs)
        u32 = ctypes.c_uint32 * n
        vp = ctypes.c_void_p * n
        i64 = ctypes.c_int64 * n
        get = lambda k: [j.get(k) for j in jobs]  # noqa: E731
        if isinstance(head, DeviceHead):
            words, head_dev, n_head = None, _p(head.words), head.n
        else:
            words = (ctypes.c_uint32 * len(head))(*[int(w) for w in head])
            head_dev, n_head = None, len(head)
        self.launches += 1
        flops = n_members * x.shape[0] * cnn.cols * sum(
            18 * a * b for a, b in zip(cnn.widths[:-1], cnn.widths[1:]))
        with self._prof("forecast", flops):
            _lib.call("enks_cnn_forward_noise", cnn.n_layers, widths, _p(cnn.w_dev), _p(cnn.b_dev),
                      float(cnn.alpha), _p(x), _ld(x), _p(u), _ld(u), _p(out), _ld(out),
                      int(x.shape[0]), int(cnn.cols), int(n_members), words, head_dev, n_head,
                      int(member0), n, u32(*[int(j["t"]) for j in jobs]),
                      u32(*[int(j["ch"]) for j in jobs]),
                      (ctypes.c_int * n)(*[int(j["rows"]) for j in jobs]),
                      vp(*[_p(v) for v in get("diag")]), vp(*[_p(v) for v in get("out")]),
                      i64(*[_ld(v) if v is not None else 0 for v in get("out")]),
                      vp(*[_p(v) for v in get("base")]),
                      i64(*[_ld(v) if v is not None else 0 for v in get("base")]),
                      vp(*[_p(v) for v in get("out_plus")]),
                      i64(*[_ld(v) if v is not None else 0 for v in get("out_plus")]),
                      self._stream())

    def burgers_forward(self, bur, x, u, out, n_members):
        """bur: engine.Forecaster of kind 'burgers' (grid, solver constants, vmax/flags)."""
        g, sub = bur.grid_n, bur.substeps
        ws = int(self.lib.enks_burgers_ws_bytes(g, int(n_members), sub))
        wsp = None
        if ws:
            if getattr(self, "_bur_ws", None) is None or self._bur_ws.numel() * 4 < ws:
                self._retire(getattr(self, "_bur_ws", None))
                self._bur_ws = torch.empty((ws + 3) // 4, dtype=torch.float32, device=self.device)
            wsp = self._bur_ws
        self.launches += 1 if not ws else sub
        _lib.call("enks_burgers_forward", _p(x), _ld(x), _p(u) if u is not None else None,
                  _ld(u) if u is not None else 0, int(u.shape[0]) if u is not None else 0,
                  _p(out), _ld(out), g, int(n_members), sub, float(bur.nu), float(bur.dt),
                  float(bur.dx), _p(bur.vmax), _p(bur.flags), _p(wsp) if wsp is not None else None,
                  self._stream())

    def barrier_row(self, bar, S, n, l, m, n_members, eps, out):
        """out (1 x n_members*m) = softplus(g(S_i)) + sqrt_var * eps_i (engine._Barrier spec)."""
        self.launches += 1
        d = n + 2 * l
        _lib.call("enks_barrier_row", _p(S), _ld(S), d, m, int(n_members), bar.kind,
                  _p(bar.coef), _ld(bar.coef) if bar.coef is not None else 0, float(bar.c0),
                  bar.r0, bar.r1, bar.alpha, bar.beta, bar.sqrt_var, _p(eps), _p(out),
                  self._stream())

    def quad_form(self, E, X, out, scale=1.0, accumulate=False):
        """out (1-element fp64 device tensor) (+)= scale * sum(E * X)."""
        self.launches += 1
        _lib.call("enks_quad_form", _p(E), _ld(E), _p(X), _ld(X), E.shape[0], E.shape[1],
                  float(scale), _p(out), int(bool(accumulate)), self._stream())

    def add(self, a, b, out):
        self.launches += 1
        _lib.call("enks_add", _p(a), _ld(a), _p(b), _ld(b), _p(out), _ld(out), out.shape[0],
                  out.shape[1], self._stream())

    def sub(self, a, b, out):
        self.launches += 1
        _lib.call("enks_sub", _p(a), _ld(a), _p(b), _ld(b), _p(out), _ld(out), out.shape[0],
                  out.shape[1], self._stream())
