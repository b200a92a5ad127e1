"""Thin Python API over the rsfde C ABI (argument marshalling only).

PyTorch provides device memory and streams; every numerical step runs in librsfde.so's
sm_100a kernels.  Names follow the ABI (and the paper): ``matvec`` (A, A~, S_alpha, H_alpha,
H_alpha^{-1}, K = P^{-1} A), ``precond`` (P_hat^{-1}, P_alpha^{-1}, P_alpha^{-1/2}),
``gmres_step``, ``solve_steps``.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _lib as L


def _dp(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(L.DP)


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr())


class RsfdeSolver:
    """One problem (d, n, alpha, kappa, tau, M, e) set up on the current CUDA device."""

    def __init__(self, d: int, n: Sequence[int], alpha: Sequence[float], kappa: Sequence[float], tau: float,
                 M: int, a_half: np.ndarray, b_half: np.ndarray, g: Sequence[Optional[np.ndarray]],
                 k: Sequence[Optional[np.ndarray]], stream=None, grid=None, grid_static: bool = False):
        """Separable e from the tables (a_half, b_half, g, k), or -- with ``grid`` (a contiguous float64
        CUDA tensor of M*N values, or N values with grid_static) -- the dense RSFDE_COEF_GRID kind."""
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("rsfde needs a CUDA device (no CPU fallback)")
        self.lib = L.load()
        self.d = d
        self.n = tuple(int(v) for v in n)
        self.M = M
        self.tau = tau
        self._keep = [np.ascontiguousarray(a_half, dtype=np.float64), np.ascontiguousarray(b_half, dtype=np.float64)]
        prob = L.rsfde_problem()
        prob.d = d
        for i in range(3):
            prob.n[i] = self.n[i] if i < d else 1
            prob.alpha[i] = alpha[i] if i < d else 2.0
            prob.kappa[i] = kappa[i] if i < d else 1.0
        prob.tau_t = tau
        prob.M = M
        prob.e.kind = L.COEF_SEPARABLE
        if grid is not None:
            if not (isinstance(grid, torch.Tensor) and grid.is_cuda and grid.dtype == torch.float64
                    and grid.is_contiguous()):
                raise TypeError("grid must be a contiguous float64 CUDA tensor")
            if grid.numel() != int(np.prod(self.n)) * (1 if grid_static else M):
                raise ValueError("grid must hold M*N values (N with grid_static)")
            self._keep.append(grid)
            prob.e.kind = L.COEF_GRID
            prob.e.grid = C.cast(C.c_void_p(grid.data_ptr()), L.DP)
            prob.e.grid_static = 1 if grid_static else 0
        prob.e.a_half = _dp(self._keep[0])
        prob.e.b_half = _dp(self._keep[1])
        for i in range(3):
            gi = g[i] if i < d else None
            ki = k[i] if i < d else None
            if gi is not None:
                gi = np.ascontiguousarray(gi, dtype=np.float64)
                self._keep.append(gi)
            if ki is not None:
                ki = np.ascontiguousarray(ki, dtype=np.float64)
                self._keep.append(ki)
            prob.e.g[i] = _dp(gi)
            prob.e.k[i] = _dp(ki)
        self._prob = prob
        ctx = C.c_void_p()
        torch.cuda.init()
        st = self.lib.rsfde_setup(C.byref(ctx), C.byref(prob), _stream(stream))
        if st != L.OK:
            raise L.RsfdeError(st, self.lib.rsfde_last_error(None).decode())
        self.ctx = ctx

    @classmethod
    def from_problem(cls, prob, stream=None) -> "RsfdeSolver":
        """Set up from a ``paper_2404_10221_b200.inputs.Problem``."""
        a_half, b_half, gs, ks = prob.e_tables()
        return cls(prob.d, prob.n, prob.alpha, prob.kappa, prob.tau, prob.M, a_half, b_half, gs, ks, stream)

    @classmethod
    def from_problem_grid(cls, prob, grid, grid_static: bool = False, stream=None) -> "RsfdeSolver":
        """Set up with the dense coefficient kind: ``grid`` holds e(x, t_{m+1/2}) on the interior grid
        for every m (M*N values) or one time-constant field (grid_static)."""
        d = prob.d
        return cls(prob.d, prob.n, prob.alpha, prob.kappa, prob.tau, prob.M, np.zeros(prob.M), np.zeros(prob.M),
                   [None] * d, [None] * d, stream, grid=grid, grid_static=grid_static)

    # ------------------------------------------------------------------ helpers
    def _check(self, st):
        if st != L.OK:
            raise L.RsfdeError(st, self.lib.rsfde_last_error(self.ctx).decode())

    def _vec(self, x):
        import torch
        if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float64 and x.is_contiguous()):
            raise TypeError("expected a contiguous float64 CUDA tensor")
        if x.numel() != int(np.prod(self.n)):
            raise ValueError(f"vector has {x.numel()} values, grid has {int(np.prod(self.n))}")
        return x

    def empty(self):
        import torch
        return torch.empty(self.n, dtype=torch.float64, device="cuda")

    # ------------------------------------------------------------------ ABI calls
    def matvec(self, op: int, x, m: int = 0, out=None, stream=None):
        x = self._vec(x)
        y = self.empty() if out is None else self._vec(out)
        self._check(self.lib.rsfde_matvec(self.ctx, op, m, _ptr(x), _ptr(y), _stream(stream)))
        return y

    def precond(self, kind: int, x, out=None, stream=None):
        x = self._vec(x)
        y = self.empty() if out is None else self._vec(out)
        self._check(self.lib.rsfde_precond_apply(self.ctx, kind, _ptr(x), _ptr(y), _stream(stream)))
        return y

    def compact_source(self, f_closed, out=None, stream=None):
        """F = (prod_l calH_l f)|interior from f on the closed grid (device tensors)."""
        import torch
        shape = tuple(v + 2 for v in self.n)
        if not (isinstance(f_closed, torch.Tensor) and f_closed.is_cuda and f_closed.dtype == torch.float64
                and f_closed.is_contiguous() and tuple(f_closed.shape) == shape):
            raise TypeError(f"expected a contiguous float64 CUDA tensor of shape {shape}")
        y = self.empty() if out is None else self._vec(out)
        self._check(self.lib.rsfde_compact_source(self.ctx, _ptr(f_closed), _ptr(y), _stream(stream)))
        return y

    @staticmethod
    def cfg(restart=50, tol=1e-9, max_iters=0, x0_policy=L.X0_PREV, form=L.FORM_A, fixed_iters=0):
        c = L.rsfde_gmres_cfg()
        c.restart, c.tol, c.max_iters = restart, tol, max_iters
        c.x0_policy, c.form, c.fixed_iters = x0_policy, form, fixed_iters
        return c

    def gmres_step(self, m: int, b, x, cfg, stream=None):
        """Solve A^{(m)} x = b in place on x (x holds x_0).  Returns (iters, relres, converged)."""
        b, x = self._vec(b), self._vec(x)
        its, rr, conv = C.c_int(), C.c_double(), C.c_int()
        self._check(self.lib.rsfde_gmres_step(self.ctx, m, _ptr(b), _ptr(x), C.byref(cfg), C.byref(its),
                                              C.byref(rr), C.byref(conv), _stream(stream)))
        return its.value, rr.value, bool(conv.value)

    def solve_steps(self, u, F=None, F_static=True, m_begin=0, m_count=None, cfg=None, stream=None):
        """March m_count CN steps in place on u (torch CUDA tensor, or numpy host array).

        F: None, one static vector, or (F_static=False) m_count stacked vectors; torch CUDA
        tensors or numpy host arrays.  Returns a report dict."""
        m_count = self.M - m_begin if m_count is None else m_count
        cfg = cfg or self.cfg()
        its = (C.c_int * max(1, m_count))()
        rr = (C.c_double * max(1, m_count))()
        cv = (C.c_ubyte * max(1, m_count))()
        rep = L.rsfde_report()
        rep.iters = its
        rep.final_relres = rr
        rep.converged = cv
        up = self._host_or_dev(u)
        Fp = None if F is None else self._host_or_dev(F)
        self._check(self.lib.rsfde_solve_steps(self.ctx, m_begin, m_count, up, Fp, 1 if F_static else 0,
                                               C.byref(cfg), C.byref(rep), _stream(stream)))
        return {"iters": list(its)[:m_count], "relres": list(rr)[:m_count],
                "converged": [bool(v) for v in cv][:m_count], "loop_seconds": rep.loop_seconds,
                "setup_seconds": rep.setup_seconds, "total_iters": rep.total_iters}

    @staticmethod
    def _host_or_dev(a):
        if isinstance(a, np.ndarray):
            if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"]:
                raise TypeError("host arrays must be C-contiguous float64")
            return C.c_void_p(a.ctypes.data)
        import torch
        if isinstance(a, torch.Tensor):
            if a.dtype != torch.float64 or not a.is_contiguous():
                raise TypeError("tensors must be contiguous float64")
            return C.c_void_p(a.data_ptr())
        raise TypeError("expected numpy array or torch tensor")

    def ebar(self):
        e, h, c = C.c_double(), C.c_double(), C.c_double()
        self._check(self.lib.rsfde_ebar(self.ctx, C.byref(e), C.byref(h), C.byref(c)))
        return e.value, h.value, c.value

    def table(self, axis: int, which: int) -> np.ndarray:
        n = self.n[axis]
        size = {0: n, 1: n, 2: n, 3: 2 * (n + 1), 4: 1}[which]
        out = np.empty(size)
        self._check(self.lib.rsfde_table(self.ctx, axis, which, out.ctypes.data_as(L.DP)))
        return out

    def profile(self, enable: bool = True) -> int:
        """Enable/disable per-launch CUDA-event timing (resets the counters)."""
        return int(self.lib.rsfde_profile(self.ctx, 1 if enable else 0))

    def profile_read(self) -> dict:
        """{class name: {"launches", "ms", "bytes"}} of the launches since rsfde_profile."""
        out = {}
        n = C.c_longlong()
        ms, by = C.c_double(), C.c_double()
        name = C.c_char_p()
        cls = 0
        while self.lib.rsfde_profile_read(self.ctx, cls, C.byref(n), C.byref(ms), C.byref(by), C.byref(name)) == 0:
            out[name.value.decode()] = {"launches": n.value, "ms": ms.value, "bytes": by.value}
            cls += 1
        return out

    def launch_count(self, reset=False) -> int:
        return int(self.lib.rsfde_launch_count(self.ctx, 1 if reset else 0))

    def graph_replays(self) -> int:
        """Replays of the graph-captured first GMRES cycle since setup (rsfde_graph_replays)."""
        return int(self.lib.rsfde_graph_replays(self.ctx))

    def device_bytes(self) -> int:
        return int(self.lib.rsfde_device_bytes(self.ctx))

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.rsfde_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_steps_batch(solvers, us, Fs=None, F_static=None, m_begin=None, m_count=None, cfgs=None):
    """rsfde_solve_steps_batch: march several independent systems concurrently (NEXT-4).

    solvers: RsfdeSolver list (distinct contexts); us: their solution vectors (torch CUDA tensors or
    numpy host arrays, updated in place); Fs / F_static / m_begin / m_count / cfgs: per-system values
    as for RsfdeSolver.solve_steps.  Returns one report dict per system."""
    B = len(solvers)
    if len(us) != B:
        raise ValueError("one u per solver")
    lib = solvers[0].lib if B else L.load()
    Fs = [None] * B if Fs is None else list(Fs)
    F_static = [True] * B if F_static is None else list(F_static)
    m_begin = [0] * B if m_begin is None else list(m_begin)
    m_count = [S.M - mb for S, mb in zip(solvers, m_begin)] if m_count is None else list(m_count)
    cfgs = [RsfdeSolver.cfg() for _ in range(B)] if cfgs is None else list(cfgs)
    ctxs = (C.c_void_p * B)(*[S.ctx.value for S in solvers])
    ub = (C.c_void_p * B)(*[RsfdeSolver._host_or_dev(u).value for u in us])
    Fb = (C.c_void_p * B)(*[None if F is None else RsfdeSolver._host_or_dev(F).value for F in Fs])
    fs = (C.c_int * B)(*[1 if f else 0 for f in F_static])
    mb = (C.c_int * B)(*m_begin)
    mc = (C.c_int * B)(*m_count)
    cf = (L.rsfde_gmres_cfg * B)(*cfgs)
    reps = (L.rsfde_report * B)()
    bufs = []
    for i in range(B):
        n = max(1, m_count[i])
        its, rr, cv = (C.c_int * n)(), (C.c_double * n)(), (C.c_ubyte * n)()
        bufs.append((its, rr, cv))
        reps[i].iters, reps[i].final_relres, reps[i].converged = its, rr, cv
    # the library's per-system streams wait for the legacy default stream only: make the inputs
    # produced on torch's current stream visible first
    import torch
    torch.cuda.current_stream().synchronize()
    st = lib.rsfde_solve_steps_batch(B, ctxs, mb, mc, ub, Fb, fs, cf, reps, None)
    if st != 0:
        msgs = [S.lib.rsfde_last_error(S.ctx).decode() for S in solvers]
        msg = next((m for m in msgs if m), "")
        raise L.RsfdeError(st, msg)
    out = []
    for i in range(B):
        its, rr, cv = bufs[i]
        k = m_count[i]
        out.append({"iters": list(its)[:k], "relres": list(rr)[:k], "converged": [bool(v) for v in cv][:k],
                    "loop_seconds": reps[i].loop_seconds, "total_iters": reps[i].total_iters})
    return out


def team_partition(n, nranks: int, rank: int):
    """rsfde_team_partition (host only, no device needed): the rank's x1 slab (layout A), x2 slab
    (layout T), the planes per rank s, s2 and the all-to-all block size in doubles."""
    lib = L.load()
    nn = (C.c_int * 3)(*[int(v) for v in n])
    out = (C.c_int * 6)()
    blk = C.c_longlong()
    st = lib.rsfde_team_partition(nn, nranks, rank, out, C.byref(blk))
    if st != L.OK:
        raise L.RsfdeError(st, "rsfde_team_partition")
    return {"x1_lo": out[0], "x1_count": out[1], "x2_lo": out[2], "x2_count": out[3], "s": out[4], "s2": out[5],
            "block": blk.value}


def team_chunking(n, nranks: int, requested: int = 0):
    """rsfde_team_chunking (host only): sub-slabs per slab, planes per sub-slab and doubles per
    (peer, chunk) piece of the chunked exchanges."""
    lib = L.load()
    nn = (C.c_int * 3)(*[int(v) for v in n])
    out = (C.c_int * 2)()
    piece = C.c_longlong()
    st = lib.rsfde_team_chunking(nn, nranks, requested, out, C.byref(piece))
    if st != L.OK:
        raise L.RsfdeError(st, "rsfde_team_chunking")
    return {"nchunk": out[0], "sc": out[1], "piece": piece.value}


class RsfdeTeam:
    """Slab-sharded 3D solver (x_1 slabs over ``nranks`` ranks).

    ``nlocal == nranks``: all ranks emulated in this process on the current device (vectors are the
    whole dense grid).  ``nlocal == 1``: one rank per process (torch.distributed / torchrun); rank 0
    creates the NCCL id (``nccl_unique_id``), the caller broadcasts it; vectors are the rank's slab
    (``slab()`` gives its x_1 range)."""

    def __init__(self, prob, nranks: int, rank: int = 0, nlocal: int = None, nccl_id: bytes = None, stream=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("rsfde needs a CUDA device (no CPU fallback)")
        self.lib = L.load()
        nlocal = nranks if nlocal is None else nlocal
        self._solo = RsfdeSolver.__new__(RsfdeSolver)  # reuse the problem marshalling
        a_half, b_half, gs, ks = prob.e_tables()
        self._keep = [np.ascontiguousarray(a_half), np.ascontiguousarray(b_half)]
        pr = L.rsfde_problem()
        pr.d = prob.d
        for i in range(3):
            pr.n[i] = prob.n[i]
            pr.alpha[i] = prob.alpha[i]
            pr.kappa[i] = prob.kappa[i]
        pr.tau_t = prob.tau
        pr.M = prob.M
        pr.e.kind = L.COEF_SEPARABLE
        pr.e.a_half = _dp(self._keep[0])
        pr.e.b_half = _dp(self._keep[1])
        for i in range(3):
            gi = None if gs[i] is None else np.ascontiguousarray(gs[i])
            ki = None if ks[i] is None else np.ascontiguousarray(ks[i])
            self._keep += [gi, ki]
            pr.e.g[i] = _dp(gi)
            pr.e.k[i] = _dp(ki)
        self._prob_struct = pr
        self.n = tuple(prob.n)
        self.M = prob.M
        self.nranks, self.rank, self.nlocal = nranks, rank, nlocal
        idbuf = None
        if nccl_id is not None:
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        t = C.c_void_p()
        st = self.lib.rsfde_team_setup(C.byref(t), C.byref(pr), nranks, rank, nlocal,
                                       None if idbuf is None else C.cast(idbuf, C.c_void_p), _stream(stream))
        if st != L.OK:
            raise L.RsfdeError(st, self.lib.rsfde_team_last_error(None).decode())
        self.team = t

    @staticmethod
    def nccl_unique_id() -> bytes:
        lib = L.load()
        buf = C.create_string_buffer(128)
        st = lib.rsfde_nccl_unique_id(C.cast(buf, C.c_void_p))
        if st != L.OK:
            raise L.RsfdeError(st, lib.rsfde_team_last_error(None).decode())
        return buf.raw

    def _check(self, st):
        if st != L.OK:
            raise L.RsfdeError(st, self.lib.rsfde_team_last_error(self.team).decode())

    def slab(self, local: int = 0):
        lo, cnt = C.c_int(), C.c_int()
        self._check(self.lib.rsfde_team_slab(self.team, local, C.byref(lo), C.byref(cnt)))
        return lo.value, cnt.value

    def local_shape(self):
        if self.nlocal == self.nranks:
            return self.n
        return (self.slab(0)[1], self.n[1], self.n[2])

    def empty(self):
        import torch
        return torch.empty(self.local_shape(), dtype=torch.float64, device="cuda")

    def matvec(self, op: int, x, m: int = 0, out=None, stream=None):
        y = self.empty() if out is None else out
        self._check(self.lib.rsfde_team_matvec(self.team, op, m, _ptr(x), _ptr(y), _stream(stream)))
        return y

    def precond(self, kind: int, x, out=None, stream=None):
        y = self.empty() if out is None else out
        self._check(self.lib.rsfde_team_precond_apply(self.team, kind, _ptr(x), _ptr(y), _stream(stream)))
        return y

    def solve_steps(self, u, F=None, F_static=True, m_begin=0, m_count=None, cfg=None, stream=None):
        m_count = self.M - m_begin if m_count is None else m_count
        cfg = cfg or RsfdeSolver.cfg()
        its = (C.c_int * max(1, m_count))()
        rr = (C.c_double * max(1, m_count))()
        cv = (C.c_ubyte * max(1, m_count))()
        rep = L.rsfde_report()
        rep.iters, rep.final_relres, rep.converged = its, rr, cv
        self._check(self.lib.rsfde_team_solve_steps(self.team, m_begin, m_count, _ptr(u),
                                                    None if F is None else _ptr(F), 1 if F_static else 0,
                                                    C.byref(cfg), C.byref(rep), _stream(stream)))
        return {"iters": list(its)[:m_count], "relres": list(rr)[:m_count],
                "converged": [bool(v) for v in cv][:m_count], "loop_seconds": rep.loop_seconds,
                "total_iters": rep.total_iters}

    def compact_source(self, f_closed_slab, local: int = 0, out=None, stream=None):
        """F on the local slab from f on the closed slab (count+2, n2+2, n3+2)."""
        lo, cnt = self.slab(local)
        y = out if out is not None else __import__("torch").empty((cnt, self.n[1], self.n[2]),
                                                                   dtype=__import__("torch").float64, device="cuda")
        self._check(self.lib.rsfde_team_compact_source(self.team, local, _ptr(f_closed_slab), _ptr(y), _stream(stream)))
        return y

    def launch_count(self, reset=False) -> int:
        return int(self.lib.rsfde_team_launch_count(self.team, 1 if reset else 0))

    def close(self):
        if getattr(self, "team", None):
            self.lib.rsfde_team_destroy(self.team)
            self.team = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
