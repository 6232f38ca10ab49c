"""paper_1509_00296_b200 — B200-native FRSVT (arXiv 1509.00296).

Thin Python binding over libfrsvt.so (C ABI in include/frsvt.h): argument
marshalling only. Every step of the hot path runs in the library's sm_100a
kernels; there is no CPU or eager-PyTorch fallback. Importing raises if the
library is missing, and every call raises on a non-OK status.

PyTorch supplies device memory, the CUDA stream and (for multi-GPU runs) the
process group used to broadcast the NCCL unique id.
"""
import ctypes
import os

import torch

from ._abi import (FRSVT_F32, FRSVT_F64, FRSVT_LMAX, FRSVT_OPT_FUSED_SKETCH, FRSVT_OPT_TF32_OMEGA, FrsvtConfig,
                   FrsvtInfo, RpcaState, load_library, status_string)

__all__ = ["Frsvt", "FrsvtError", "LoopbackGroup", "batched_apply", "lib", "library_path", "colmajor", "W_EXPLICIT",
           "W_RECIPROCAL", "W_REWEIGHTED", "FRSVT_OPT_FUSED_SKETCH", "FRSVT_OPT_TF32_OMEGA", "FLAG_NONFINITE",
           "FLAG_NOCONV", "FLAG_NONMONOTONE_W", "FLAG_SINGLE_CTA"]

W_EXPLICIT, W_RECIPROCAL, W_REWEIGHTED = 0, 1, 2
# frsvt_info.flags bits (include/frsvt.h FRSVT_FLAG_*)
FLAG_NONFINITE, FLAG_NOCONV, FLAG_NONMONOTONE_W, FLAG_SINGLE_CTA = 1, 2, 4, 8

lib, library_path = load_library()


class FrsvtError(RuntimeError):
    def __init__(self, fn, st):
        super().__init__("%s failed: %s (status %d)" % (fn, status_string(lib, st), st))
        self.status = st


def _check(fn, st):
    if st != 0:
        raise FrsvtError(fn, st)


def colmajor(x):
    """Column-major copy/view of a 2-D tensor (the library layout)."""
    if x.stride(0) == 1 and x.stride(1) >= max(1, x.shape[0]):
        return x
    return x.t().contiguous().t()


def _ld(x, rows, dtype, name):
    if x.device.type != "cuda":
        raise ValueError("%s must be a CUDA tensor" % name)
    if x.dtype != dtype:
        raise ValueError("%s must be %s, got %s" % (name, dtype, x.dtype))
    if x.dim() != 2 or x.shape[0] != rows:
        raise ValueError("%s must have %d rows, got shape %s" % (name, rows, tuple(x.shape)))
    if x.stride(0) != 1 or x.stride(1) < max(1, rows):
        raise ValueError("%s must be column-major (stride (1, ld>=rows)), got %s" % (name, x.stride()))
    return x.stride(1)


def batched_apply(A, Omega, q=1, tau=None, w=None, stream=None, X=None):
    """frsvt_batched_apply (fp32) / frsvt_batched_apply_f64 (fp64): X[b] =
    FRSVT(A[b]) for a batch of small matrices (one CTA each). A: (batch, m, n)
    CUDA fp32 or fp64 with each matrix column-major (A[b].stride() == (1, ld));
    Omega: n x l column-major. tau: a float or a (batch,) tensor; w: (l,)
    weights. X (optional): the output, (batch, m, n) of A's dtype with
    column-major matrices (any ld >= m, any batch stride); allocated when None.
    Returns X, r (batch,) int32, sigma (batch, l) float64."""
    if A.dim() != 3 or A.dtype not in (torch.float32, torch.float64) or A.device.type != "cuda":
        raise ValueError("A must be a (batch, m, n) CUDA fp32 or fp64 tensor")
    dt = A.dtype
    batch, m, n = A.shape
    if batch == 0:
        l = Omega.shape[1]
        return (torch.empty((0, m, n), dtype=dt, device=A.device),
                torch.empty(0, dtype=torch.int32, device=A.device),
                torch.empty((0, l), dtype=torch.float64, device=A.device))
    if A.stride(1) != 1:
        raise ValueError("each A[b] must be column-major")
    lda, sA = A.stride(2), A.stride(0)
    Om = colmajor(Omega.to(device=A.device, dtype=dt))
    l = Om.shape[1]
    if X is None:
        X = torch.empty((batch, n, m), dtype=dt, device=A.device).transpose(1, 2)
    elif (X.shape != A.shape or X.dtype != dt or X.device != A.device or X.stride(1) != 1
          or X.stride(2) < max(1, m)):
        raise ValueError("X must be a (batch, m, n) tensor of A's dtype on A's device with column-major matrices")
    r = torch.empty(batch, dtype=torch.int32, device=A.device)
    sig = torch.empty((batch, l), dtype=torch.float64, device=A.device)
    wmode, tau_s, tau_p, w_p = 0, 0.0, None, None
    if w is not None:
        wmode = 1
        wt = torch.as_tensor(w, dtype=torch.float64, device=A.device).contiguous()
        w_p = ctypes.c_void_p(wt.data_ptr())
    elif torch.is_tensor(tau):
        tt = tau.to(device=A.device, dtype=torch.float64).contiguous()
        tau_p = ctypes.c_void_p(tt.data_ptr())
    else:
        tau_s = float(tau)
    st = stream if stream is not None else torch.cuda.current_stream()
    for t in (A, Om, X) + ((wt,) if w is not None else ()) + ((tt,) if tau_p is not None else ()):
        t.record_stream(st)  # kept alive for the asynchronous kernel on `st`
    name = "frsvt_batched_apply" if dt == torch.float32 else "frsvt_batched_apply_f64"
    _check(name, getattr(lib, name)(
        int(batch), int(m), int(n), int(l), int(q), ctypes.c_void_p(A.data_ptr()), int(lda), int(sA),
        ctypes.c_void_p(Om.data_ptr()), int(Om.stride(1)), wmode, tau_s, tau_p, w_p, ctypes.c_void_p(X.data_ptr()),
        int(X.stride(2)), int(X.stride(0)), ctypes.c_void_p(r.data_ptr()), ctypes.c_void_p(sig.data_ptr()),
        ctypes.c_void_p(st.cuda_stream)))
    return X, r, sig


class LoopbackGroup:
    """frsvt_loopback_create: `nranks` virtual ranks of the row-sharded path on
    one device, one handle (Frsvt(..., group=g)) and host thread per rank."""

    def __init__(self, nranks):
        self._g = ctypes.c_void_p()
        self.nranks = int(nranks)
        _check("frsvt_loopback_create", lib.frsvt_loopback_create(self.nranks, ctypes.byref(self._g)))

    @property
    def ptr(self):
        return self._g

    def close(self):
        if self._g.value:
            lib.frsvt_loopback_destroy(self._g)
            self._g = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Frsvt:
    """One FRSVT handle: fixed shape (m_local x n), sketch width l, power
    iterations q, range propagation flag, dtype (torch.float32/float64)."""

    def __init__(self, m, n, l, q=1, rp=True, dtype=torch.float32, seed=0, stream=None,
                 nranks=1, rank=0, m_global=None, row0=0, nccl_id=None, device=None, options=0, group=None):
        if device is not None:
            torch.cuda.set_device(device)
        self.m, self.n, self.l, self.q, self.rp = int(m), int(n), int(l), int(q), bool(rp)
        self.dtype = dtype
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        cfg = FrsvtConfig()
        cfg.dtype = FRSVT_F32 if dtype == torch.float32 else FRSVT_F64
        cfg.m_local = self.m
        cfg.n = self.n
        cfg.m_global = self.m if m_global is None else int(m_global)
        cfg.row0 = int(row0)
        cfg.l = self.l
        cfg.q = self.q
        cfg.range_propagation = 1 if rp else 0
        cfg.seed = int(seed)
        cfg.nranks = int(nranks)
        cfg.rank = int(rank)
        cfg.options = int(options)
        self._group = group
        if group is not None:
            cfg.group = group.ptr.value
        self._id_buf = None
        if nccl_id is not None:
            self._id_buf = (ctypes.c_ubyte * 128)(*bytes(nccl_id))
            cfg.nccl_id = ctypes.cast(self._id_buf, ctypes.POINTER(ctypes.c_ubyte))
        self._h = ctypes.c_void_p()
        _check("frsvt_create", lib.frsvt_create(ctypes.byref(cfg), ctypes.c_void_p(self.stream.cuda_stream),
                                                ctypes.byref(self._h)))
        self.cfg = cfg

    # -- lifecycle --------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib.frsvt_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def unique_id():
        buf = (ctypes.c_ubyte * 128)()
        _check("frsvt_get_unique_id", lib.frsvt_get_unique_id(buf))
        return bytes(buf)

    # -- operator ---------------------------------------------------------
    def _out(self, X, like):
        if X is None:
            X = torch.empty((self.n, self.m), dtype=self.dtype, device=like.device).t()
        return X

    def apply(self, A, tau, X=None, info=False):
        """X = FRSVT_tau(A) (Alg. 1, Eq. 6). Returns X (and FrsvtInfo if info)."""
        lda = _ld(A, self.m, self.dtype, "A")
        X = self._out(X, A)
        ldx = _ld(X, self.m, self.dtype, "X")
        inf = FrsvtInfo() if info else None
        _check("frsvt_apply", lib.frsvt_apply(self._h, ctypes.c_void_p(A.data_ptr()), lda, float(tau),
                                              ctypes.c_void_p(X.data_ptr()), ldx,
                                              ctypes.byref(inf) if info else None))
        return (X, inf) if info else X

    def apply_weighted(self, A, mode, w=None, C=0.0, eps=1e-6, X=None, info=False):
        """Weighted SVT: mode W_EXPLICIT (w, length l), W_RECIPROCAL
        (C/(sigma+eps)) or W_REWEIGHTED (C/(d_prev+eps))."""
        lda = _ld(A, self.m, self.dtype, "A")
        X = self._out(X, A)
        ldx = _ld(X, self.m, self.dtype, "X")
        wbuf = None
        if mode == W_EXPLICIT:
            if w is None or len(w) < self.l:
                raise ValueError("explicit weights need l values")
            wbuf = (ctypes.c_double * self.l)(*[float(v) for v in list(w)[: self.l]])
        inf = FrsvtInfo() if info else None
        _check("frsvt_apply_weighted",
               lib.frsvt_apply_weighted(self._h, ctypes.c_void_p(A.data_ptr()), lda, int(mode), wbuf,
                                        float(C), float(eps), ctypes.c_void_p(X.data_ptr()), ldx,
                                        ctypes.byref(inf) if info else None))
        return (X, inf) if info else X

    def rpca_step(self, state, finalize=False, want_resid=False):
        """One fused iALM step (rpca_alm_step). `state` is an RpcaState."""
        res = ctypes.c_double(0.0)
        _check("rpca_alm_step", lib.rpca_alm_step(self._h, ctypes.byref(state), 1 if finalize else 0,
                                                  ctypes.byref(res) if want_resid else None))
        return res.value if want_resid else None

    def rpca_state(self, D, E, A, L=None, lam=0.0, rho=1.5, mu_max_factor=1e7, norm2_D=0.0, mu0=0.0, keep=0,
                   transfer=False):
        ld = _ld(D, self.m, self.dtype, "D")
        for t, nm in ((E, "E"), (A, "A")) + (((L, "L"),) if L is not None else ()):
            if _ld(t, self.m, self.dtype, nm) != ld:
                raise ValueError("D, E, A, L must share one leading dimension")
        st = RpcaState()
        st.D = D.data_ptr()
        st.E = E.data_ptr()
        st.A = A.data_ptr()
        st.L = L.data_ptr() if L is not None else None
        st.ld = ld
        st.lambda_ = float(lam)
        st.rho = float(rho)
        st.mu_max_factor = float(mu_max_factor)
        st.norm2_D = float(norm2_D)
        st.mu0 = float(mu0)
        st.iter = 0
        st.keep = int(keep)
        st.transfer = 1 if transfer else 0
        st._keep = (D, E, A, L)
        return st

    # -- hooks ------------------------------------------------------------
    def set_omega(self, Om):
        ld = _ld(Om, self.n, self.dtype, "Omega")
        _check("frsvt_set_omega", lib.frsvt_set_omega(self._h, ctypes.c_void_p(Om.data_ptr()), ld))

    def draw_omega(self, call):
        out = torch.empty((self.l, self.n), dtype=self.dtype, device="cuda").t()
        _check("frsvt_draw_omega", lib.frsvt_draw_omega(self._h, int(call), ctypes.c_void_p(out.data_ptr()),
                                                        self.n))
        return out

    def get_carry(self):
        out = torch.empty((self.l, self.m), dtype=self.dtype, device="cuda").t()
        r = ctypes.c_int32(0)
        _check("frsvt_get_carry", lib.frsvt_get_carry(self._h, ctypes.c_void_p(out.data_ptr()), self.m,
                                                      ctypes.byref(r)))
        return out[:, : r.value], r.value

    def set_carry(self, Qt):
        r = 0 if Qt is None else Qt.shape[1]
        if r:
            Qt = colmajor(Qt.to(self.dtype).cuda())
            ld = _ld(Qt, self.m, self.dtype, "carry")
            ptr = ctypes.c_void_p(Qt.data_ptr())
        else:
            ld, ptr = self.m, None
        _check("frsvt_set_carry", lib.frsvt_set_carry(self._h, ptr, ld, r))

    def reset_carry(self):
        _check("frsvt_reset_carry", lib.frsvt_reset_carry(self._h))

    def set_adaptive_rank(self, a=2, p_jump=None, b=None, l0=None, rho=0.05, gamma=None):
        """Adaptive rank prediction (Eq. 7): a, p_jump = ceil(rho n_min) (the
        jump when the kept rank fills the sketch), bound b (default l, or
        ceil(gamma n_min)), l0 (default ceil(0.1 b)). a=0 switches it off."""
        import math
        nmin = min(self.cfg.m_global, self.n)
        if b is None:
            b = self.l if gamma is None else min(self.l, int(math.ceil(gamma * nmin)))
        if p_jump is None:
            p_jump = max(1, int(math.ceil(rho * nmin)))
        if l0 is None:
            l0 = max(1, int(math.ceil(0.1 * b)))
        _check("frsvt_set_adaptive_rank", lib.frsvt_set_adaptive_rank(self._h, int(a), int(p_jump), int(b), int(l0)))
        return dict(a=a, rho_n=p_jump, b=b, l0=l0)

    def set_call_index(self, call):
        _check("frsvt_set_call_index", lib.frsvt_set_call_index(self._h, int(call)))

    def info(self):
        inf = FrsvtInfo()
        _check("frsvt_get_info", lib.frsvt_get_info(self._h, ctypes.byref(inf)))
        return inf

    def get_mu(self):
        v = ctypes.c_double(0.0)
        _check("rpca_get_mu", lib.rpca_get_mu(self._h, ctypes.byref(v)))
        return v.value

    def set_mu(self, mu, mu_bar):
        _check("rpca_set_mu", lib.rpca_set_mu(self._h, float(mu), float(mu_bar)))

    def debug_pass(self, kind, impl, A, B):
        """kind 0: A @ B (m x l); kind 1: A.T @ B (n x l). impl 0 SIMT, 1 tcgen05."""
        lda = _ld(A, self.m, self.dtype, "A")
        if kind == 0:
            B = colmajor(B)
            _ld(B, self.n, self.dtype, "B")
            out = torch.empty((self.l, self.m), dtype=self.dtype, device=A.device).t()
        else:
            B = colmajor(B)
            _ld(B, self.m, self.dtype, "B")
            out = torch.empty((self.l, self.n), dtype=self.dtype, device=A.device).t()
        if B.stride(1) != B.shape[0]:
            B = B.t().contiguous().t()
        _check("frsvt_debug_pass", lib.frsvt_debug_pass(self._h, int(kind), int(impl), ctypes.c_void_p(A.data_ptr()),
                                                        lda, ctypes.c_void_p(B.data_ptr()),
                                                        ctypes.c_void_p(out.data_ptr())))
        return out

    def debug_small_svd(self, impl=0, G=None, reps=0):
        """Small SVD of an l x l fp64 Gram (None = the last call's Gram).
        Returns (sigma, UB, G_used, sweeps, mean_ms)."""
        l = self.l
        dev = torch.device("cuda", torch.cuda.current_device())
        if G is not None:
            G = G.to(device=dev, dtype=torch.float64).t().contiguous().t()
            if tuple(G.shape) != (l, l):
                raise ValueError("G must be %d x %d" % (l, l))
        Gc = torch.empty((l, l), dtype=torch.float64, device=dev).t()
        sig = torch.empty(l, dtype=torch.float64, device=dev)
        UB = torch.empty((l, l), dtype=torch.float64, device=dev).t()
        sw, ms = ctypes.c_int32(), ctypes.c_double()
        _check("frsvt_debug_small_svd", lib.frsvt_debug_small_svd(
            self._h, int(impl), ctypes.c_void_p(G.data_ptr() if G is not None else 0),
            ctypes.c_void_p(Gc.data_ptr()), ctypes.c_void_p(sig.data_ptr()), ctypes.c_void_p(UB.data_ptr()),
            ctypes.byref(sw), int(reps), ctypes.byref(ms)))
        return sig, UB, Gc, sw.value, ms.value

    def debug_pass_timed(self, kind, impl, A, B, reps=10):
        """Mean device ms of `reps` back-to-back passes (see debug_pass)."""
        lda = _ld(A, self.m, self.dtype, "A")
        B = colmajor(B)
        rows = self.n if kind == 0 else self.m
        _ld(B, rows, self.dtype, "B")
        if B.stride(1) != B.shape[0]:
            B = B.t().contiguous().t()
        out = torch.empty((self.l, self.m if kind == 0 else self.n), dtype=self.dtype, device=A.device).t()
        ms = ctypes.c_double()
        _check("frsvt_debug_pass_timed", lib.frsvt_debug_pass_timed(
            self._h, int(kind), int(impl), ctypes.c_void_p(A.data_ptr()), lda, ctypes.c_void_p(B.data_ptr()),
            ctypes.c_void_p(out.data_ptr()), int(reps), ctypes.byref(ms)))
        return ms.value

    def debug_chol(self, G, stamps=False):
        """CholeskyQR factor T of an l x l Gram; returns (T, s[, stamps ns])."""
        l = self.l
        dev = torch.device("cuda", torch.cuda.current_device())
        G = G.to(device=dev, dtype=torch.float64).t().contiguous().t()
        T = torch.empty((l, l), dtype=self.dtype, device=dev).t()
        st = torch.zeros(8, dtype=torch.int64, device=dev) if stamps else None
        s = ctypes.c_int32()
        _check("frsvt_debug_chol", lib.frsvt_debug_chol(self._h, ctypes.c_void_p(G.data_ptr()),
                                                        ctypes.c_void_p(T.data_ptr()), ctypes.byref(s),
                                                        ctypes.c_void_p(st.data_ptr() if st is not None else 0)))
        return (T, s.value, st.cpu().numpy()) if stamps else (T, s.value)

    def debug_chol_inv(self, G, r=0, stamps=False):
        """Explicit CholeskyQR factor (chol_inv.cuh) of an l x l Gram whose first
        r columns are orthonormal; returns (T fp32 l x l, s[, stamps ns])."""
        l = self.l
        dev = torch.device("cuda", torch.cuda.current_device())
        G = G.to(device=dev, dtype=torch.float64).t().contiguous().t()
        T = torch.empty((l, l), dtype=torch.float32, device=dev).t()
        st = torch.zeros(8, dtype=torch.int64, device=dev) if stamps else None
        s = ctypes.c_int32()
        _check("frsvt_debug_chol_inv", lib.frsvt_debug_chol_inv(
            self._h, ctypes.c_void_p(G.data_ptr()), int(r), ctypes.c_void_p(T.data_ptr()), ctypes.byref(s),
            ctypes.c_void_p(st.data_ptr() if st is not None else 0)))
        return (T, s.value, st.cpu().numpy()) if stamps else (T, s.value)

    def profile(self, enable=True):
        _check("frsvt_profile", lib.frsvt_profile(self._h, 1 if enable else 0))

    def profile_read(self):
        """{kind: (ms, launches, bytes)} for kinds 'AX', 'AtQ', 'compose', and
        'single' (single-CTA calls; the third value is their FLOP count)."""
        out = {}
        for k, name in enumerate(("AX", "AtQ", "compose", "single")):
            ms, n, b = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double()
            _check("frsvt_profile_read", lib.frsvt_profile_read(self._h, k, ctypes.byref(ms), ctypes.byref(n),
                                                                ctypes.byref(b)))
            out[name] = (ms.value, n.value, b.value)
        return out

    @property
    def launches(self):
        return int(lib.frsvt_kernel_launches(self._h))
