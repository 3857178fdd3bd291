"""Thin Python binding of librotvote (include/rotvote.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of ``librotvote.so``; this
module converts torch tensors to raw pointers and C structs to Python objects.
It raises ``ImportError`` when the extension is missing -- there is no CPU or
PyTorch fallback.

Names follow the C-ABI: ``rot_vote_create``, ``rot_vote_solve``,
``rot_vote_solve_batched`` ... plus a small ``RotVote`` convenience class.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RV_LIB") or os.path.join(_HERE, "librotvote.so")  # RV_LIB: tuning variants

RV_OK, RV_EINVAL, RV_EDATA, RV_ECUDA, RV_ENCCL, RV_ENOMEM = 0, -1, -2, -3, -4, -5
RV_REFINED, RV_DEGENERATE, RV_RECHECKED = 1, 2, 4
RV_MODE_BOUND, RV_MODE_FINAL, RV_MODE_EXACT, RV_MODE_BOUND_TC, RV_MODE_FINAL_TC = 0, 1, 2, 3, 4
RV_MAX_CHAIN, RV_MAX_PHASES = 8, 16
DEFAULT_CHAIN = (5, 15, 45, 90, 180, 360)

_ERRNAMES = {RV_EINVAL: "RV_EINVAL", RV_EDATA: "RV_EDATA", RV_ECUDA: "RV_ECUDA",
             RV_ENCCL: "RV_ENCCL", RV_ENOMEM: "RV_ENOMEM"}


class RotVoteError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_ERRNAMES.get(code, code)}: {msg}")
        self.code = code


class rv_config(C.Structure):
    _fields_ = [("device", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
                ("nccl_id", C.c_void_p), ("max_n", C.c_int64), ("max_problems", C.c_int32),
                ("chain_len", C.c_int32), ("chain", C.c_int32 * RV_MAX_CHAIN),
                ("refine_rounds", C.c_int32), ("guard", C.c_float), ("stream", C.c_void_p),
                ("emulate_world", C.c_int32), ("tensor_vote", C.c_int32), ("cull", C.c_int32),
                ("planner", C.c_int32), ("ct_sched", C.c_int32)]


class rv_result(C.Structure):
    _fields_ = [("q", C.c_double * 4), ("q_cell", C.c_double * 4), ("votes", C.c_uint32),
                ("n_inliers", C.c_uint32), ("cell", C.c_int32 * 3), ("flags", C.c_int32),
                ("B", C.c_int32), ("n_tied", C.c_int32), ("pair_votes", C.c_uint64),
                ("cells_evaluated", C.c_uint64), ("lb_star", C.c_uint32), ("n_phases", C.c_int32),
                ("cells_per_phase", C.c_int64 * RV_MAX_PHASES), ("ms", C.c_float),
                ("n_rechecked", C.c_int32), ("vote_ms", C.c_float), ("launches", C.c_int32),
                ("vote_pairs", C.c_uint64), ("vote_launches", C.c_int32),
                ("cull_launches", C.c_int32), ("cull_pairs", C.c_uint64), ("cull_ms", C.c_float),
                ("cull_tc_launches", C.c_int32), ("host_syncs", C.c_int32),
                ("t_setup_ms", C.c_float), ("t_level0_ms", C.c_float), ("t_dive_ms", C.c_float),
                ("t_bnb_ms", C.c_float), ("t_final_ms", C.c_float), ("t_refine_ms", C.c_float)]


class rv_alg1_result(C.Structure):
    _fields_ = [("q", C.c_double * 4), ("votes", C.c_uint32), ("cell", C.c_int32 * 3),
                ("B", C.c_int32), ("J", C.c_int32), ("samples", C.c_uint64), ("ms", C.c_float),
                ("vote_ms", C.c_float)]


class rv_rigid_result(C.Structure):
    _fields_ = [("q", C.c_double * 4), ("t", C.c_double * 3), ("t_mean", C.c_double * 3),
                ("rot_votes", C.c_uint32), ("rot_inliers", C.c_uint32), ("t_votes", C.c_uint32),
                ("t_cell", C.c_int32 * 3), ("pad_", C.c_int32), ("pairs_total", C.c_int64),
                ("pairs_kept", C.c_int64), ("ms", C.c_float), ("pairs_ms", C.c_float),
                ("rot_ms", C.c_float), ("trans_ms", C.c_float)]


class rv_plan_result(C.Structure):
    _fields_ = [("lin", C.c_uint32), ("B", C.c_int32), ("votes", C.c_uint32), ("n_tied", C.c_int32),
                ("lb_star", C.c_uint32), ("n_rechecked", C.c_int32), ("pair_votes", C.c_uint64),
                ("cells_evaluated", C.c_uint64), ("n_phases", C.c_int32),
                ("cells_per_phase", C.c_int64 * 16)]


_lib = None


def lib() -> C.CDLL:
    """Load librotvote.so (raises ImportError if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"librotvote.so not built at {LIB_PATH}: run "
                          "`python -m paper_2506_11547_b200.build` (or __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    vp, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_double
    L.rot_vote_default_config.argtypes = [C.POINTER(rv_config)]
    L.rot_vote_default_config.restype = None
    L.rot_vote_create.argtypes = [C.POINTER(rv_config), C.POINTER(vp)]
    L.rot_vote_destroy.argtypes = [vp]
    L.rot_vote_destroy.restype = None
    L.rot_vote_last_error.argtypes = [vp]
    L.rot_vote_last_error.restype = C.c_char_p
    L.rot_vote_get_unique_id.argtypes = [vp]
    L.rot_vote_solve.argtypes = [vp, vp, vp, i64, dbl, i32, C.POINTER(rv_result), vp]
    L.rot_vote_solve_host.argtypes = [vp, vp, vp, i64, dbl, i32, C.POINTER(rv_result), vp]
    L.rot_vote_solve_batched.argtypes = [vp, vp, vp, vp, i32, dbl, i32, C.POINTER(rv_result), vp]
    L.rot_vote_setup.argtypes = [vp, vp, vp, i64, vp]
    L.rot_vote_count_cells.argtypes = [vp, vp, vp, i64, i32, vp, i64, dbl, i32, vp, vp]
    L.rot_vote_refine.argtypes = [vp, vp, vp, i64, dbl, vp, i32, vp, vp, vp, vp]
    L.rot_vote_alg1.argtypes = [vp, vp, vp, i64, i32, C.POINTER(rv_alg1_result), vp]
    L.rot_vote_rigid.argtypes = [vp, vp, vp, i64, dbl, dbl, i32, dbl, dbl, dbl,
                                 C.POINTER(rv_rigid_result), vp, i64]
    L.rot_vote_translation.argtypes = [vp, vp, vp, i64, vp, dbl, dbl, dbl, C.POINTER(i64),
                                       C.POINTER(C.c_uint32), vp, vp]
    L.rot_vote_solve_multi.argtypes = [vp, vp, vp, i64, dbl, i32, i32, dbl, C.POINTER(rv_result),
                                       C.POINTER(i32)]
    L.rot_vote_debug_tc_scores.argtypes = [vp, vp, vp, i64, i32, vp, i64, dbl, vp]
    L.rot_vote_count_cells_culled.argtypes = [vp, vp, vp, i64, i32, i32, vp, i64, dbl, i32, vp, vp,
                                              vp]
    L.rv_plan_request_is_full_grid.argtypes = [vp]
    L.rv_plan_create.argtypes = [vp, i32, i32, i64, dbl, dbl, C.POINTER(vp)]
    L.rv_plan_create_ex.argtypes = [vp, i32, i32, i64, dbl, dbl, vp, i32, dbl, C.POINTER(vp)]
    L.rv_plan_destroy.argtypes = [vp]
    L.rv_plan_destroy.restype = None
    L.rv_plan_request.argtypes = [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i64),
                                  C.POINTER(C.POINTER(C.c_uint32))]
    L.rv_plan_feed.argtypes = [vp, vp, vp]
    L.rv_plan_get_result.argtypes = [vp, C.POINTER(rv_plan_result)]
    L.rv_shard_range.argtypes = [i64, i32, i32, C.POINTER(i64), C.POINTER(i64)]
    L.rv_shard_range.restype = None
    L.rv_grid_candidates.argtypes = [i32, vp, i64]
    L.rv_grid_candidates.restype = i64
    L.rv_cull_groups.argtypes = [i32, i32, i32, i32, vp, vp, vp]
    L.rv_cull_groups.restype = i64
    L.rv_cull_partition.argtypes = [i32, i32, i32, i32, i32, vp, vp]
    L.rv_cull_partition.restype = i32
    _lib = L
    return L


# ---- plain C-ABI wrappers ----------------------------------------------------------------

def rot_vote_default_config() -> rv_config:
    cfg = rv_config()
    lib().rot_vote_default_config(C.byref(cfg))
    return cfg


def rot_vote_get_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    rc = lib().rot_vote_get_unique_id(buf)
    if rc != RV_OK:
        raise RotVoteError(rc, "ncclGetUniqueId failed (libnccl.so.2 not loadable?)")
    return buf.raw


def rot_vote_create(cfg: rv_config) -> int:
    h = C.c_void_p()
    rc = lib().rot_vote_create(C.byref(cfg), C.byref(h))
    if rc != RV_OK:
        raise RotVoteError(rc, "rot_vote_create failed")
    return h.value


def rot_vote_destroy(ctx: int) -> None:
    lib().rot_vote_destroy(ctx)


def _check(ctx, rc):
    if rc != RV_OK:
        raise RotVoteError(rc, lib().rot_vote_last_error(ctx).decode())


def _dptr(t, dtype, name):
    """Device pointer of a contiguous CUDA tensor of the given torch dtype."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous {dtype} tensor")
    return t.data_ptr()


PHASES = ("setup", "level0", "dive", "bnb", "final", "refine")
RV_RETRIED = 8


@dataclass
class Result:
    q: np.ndarray
    q_cell: np.ndarray
    votes: int
    n_inliers: int
    cell: tuple
    flags: int
    B: int
    n_tied: int
    pair_votes: int
    cells_evaluated: int
    lb_star: int
    cells_per_phase: list
    ms: float
    n_rechecked: int
    vote_ms: float = 0.0
    launches: int = 0
    vote_pairs: int = 0
    vote_launches: int = 0
    cull_launches: int = 0
    cull_pairs: int = 0
    cull_ms: float = 0.0
    cull_tc_launches: int = 0
    host_syncs: int = 0
    phase_ms: dict = None   # one-pass solves: device time per phase (CUDA events)

    @property
    def lin(self) -> int:
        i, j, k = self.cell
        return (i * self.B + j) * self.B + k

    @staticmethod
    def from_c(r: rv_result) -> "Result":
        return Result(q=np.array(r.q[:]), q_cell=np.array(r.q_cell[:]), votes=r.votes,
                      n_inliers=r.n_inliers, cell=tuple(r.cell[:]), flags=r.flags, B=r.B,
                      n_tied=r.n_tied, pair_votes=r.pair_votes, cells_evaluated=r.cells_evaluated,
                      lb_star=r.lb_star, cells_per_phase=list(r.cells_per_phase[:r.n_phases]),
                      ms=r.ms, n_rechecked=r.n_rechecked, vote_ms=r.vote_ms,
                      launches=r.launches, vote_pairs=r.vote_pairs,
                      vote_launches=r.vote_launches, cull_launches=r.cull_launches,
                      cull_pairs=r.cull_pairs, cull_ms=r.cull_ms,
                      cull_tc_launches=r.cull_tc_launches, host_syncs=r.host_syncs,
                      phase_ms={k: getattr(r, f"t_{k}_ms") for k in PHASES})


class RotVote:
    """A librotvote context bound to one CUDA device and stream."""

    def __init__(self, device: int = 0, max_n: int = 1 << 20, max_problems: int = 1,
                 chain=None, refine_rounds: int = 2, guard: float = 1e-5, stream=None,
                 rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 emulate_world: int = 0, tensor_vote: bool = True, cull=True,
                 planner: str = "device", ct_sched: str = "auto"):
        """cull: True / "tc" (K3-CT, default), "fp32" (K3-C), False (off).
        planner: "device" (the level loop on the GPU, one host round trip per single solve;
        default), "device_sync" (the device loop with a round trip per level, the one-pass
        solve's fallback) or "host" (rv_plan.cpp)."""
        import torch
        self._kw = dict(device=device, max_n=max_n, max_problems=max_problems, chain=chain,
                        refine_rounds=refine_rounds, guard=guard, stream=stream, rank=rank,
                        world=world, nccl_id=nccl_id, emulate_world=emulate_world,
                        tensor_vote=tensor_vote, cull=cull, planner=planner, ct_sched=ct_sched)
        cfg = rot_vote_default_config()
        cfg.device = device
        cfg.rank, cfg.world = rank, world
        self._id_buf = None
        if nccl_id is not None:
            self._id_buf = C.create_string_buffer(nccl_id, 128)
            cfg.nccl_id = C.cast(self._id_buf, C.c_void_p)
        cfg.max_n = int(max_n)
        cfg.max_problems = int(max_problems)
        if chain is not None:
            cfg.chain_len = len(chain)
            for a, b in enumerate(chain):
                cfg.chain[a] = int(b)
        cfg.refine_rounds = int(refine_rounds)
        cfg.guard = float(guard)
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        cfg.stream = C.c_void_p(stream.cuda_stream)
        cfg.emulate_world = int(emulate_world)
        cfg.tensor_vote = int(bool(tensor_vote))
        cfg.cull = {True: 1, "tc": 1, "fp32": 2, False: 0, None: 0}[cull]
        cfg.planner = {"device": 0, "host": 1, "device_sync": 2}[planner]
        cfg.ct_sched = {"auto": 0, "static": 1}[ct_sched]
        self.cfg = cfg
        self.device = device
        self.chain = tuple(chain) if chain is not None else DEFAULT_CHAIN
        self.ctx = rot_vote_create(cfg)

    def twin(self, **overrides) -> "RotVote":
        """A second context with this one's settings, some overridden (e.g. planner="host")."""
        return RotVote(**{**self._kw, **overrides})

    def close(self):
        if getattr(self, "ctx", None):
            rot_vote_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def last_error(self) -> str:
        return lib().rot_vote_last_error(self.ctx).decode()

    # -- hot path --
    def solve(self, x, y, eps: float, levels: int = 0, mask=None) -> Result:
        import torch
        n = x.shape[0]
        r = rv_result()
        mp = _dptr(mask, torch.int32, "mask") if mask is not None else None
        _check(self.ctx, lib().rot_vote_solve(self.ctx, _dptr(x, torch.float32, "x"),
                                              _dptr(y, torch.float32, "y"), n, float(eps),
                                              int(levels), C.byref(r), mp))
        return Result.from_c(r)

    def solve_host(self, x: np.ndarray, y: np.ndarray, eps: float, levels: int = 0,
                   mask: np.ndarray | None = None) -> Result:
        x = np.ascontiguousarray(x, np.float32)
        y = np.ascontiguousarray(y, np.float32)
        r = rv_result()
        mp = None
        if mask is not None:
            assert mask.dtype == np.uint32 and mask.flags.c_contiguous
            mp = mask.ctypes.data
        _check(self.ctx, lib().rot_vote_solve_host(self.ctx, x.ctypes.data, y.ctypes.data,
                                                   x.shape[0], float(eps), int(levels),
                                                   C.byref(r), mp))
        return Result.from_c(r)

    def solve_batched(self, x, y, offsets, eps: float, levels: int = 0, masks=None,
                      raw: bool = False):
        """P independent problems (rows offsets[p]..offsets[p+1] of x / y).  Returns a list of
        Result, or with raw=True the rv_result array itself as a numpy structured array
        (fields as in include/rotvote.h; no per-problem Python objects)."""
        import torch
        offs = np.ascontiguousarray(offsets, np.int64)
        P = offs.size - 1
        out = (rv_result * P)()
        mp = _dptr(masks, torch.int32, "masks") if masks is not None else None
        _check(self.ctx, lib().rot_vote_solve_batched(
            self.ctx, _dptr(x, torch.float32, "x"), _dptr(y, torch.float32, "y"),
            offs.ctypes.data, P, float(eps), int(levels), out, mp))
        if raw:
            return np.ctypeslib.as_array(out)
        return [Result.from_c(out[p]) for p in range(P)]

    # -- individual steps (parity tests) --
    def setup(self, x, y):
        import torch
        n = x.shape[0]
        k = torch.empty((9, n), dtype=torch.float32, device=x.device)
        _check(self.ctx, lib().rot_vote_setup(self.ctx, _dptr(x, torch.float32, "x"),
                                              _dptr(y, torch.float32, "y"), n, k.data_ptr()))
        return k

    def count_cells(self, x, y, B: int, lins, eps: float, mode: int):
        import torch
        lins = torch.as_tensor(np.asarray(lins, np.uint32).view(np.int32), device=x.device)
        m = lins.numel()
        a = torch.zeros(m, dtype=torch.int32, device=x.device)
        b = torch.zeros(m, dtype=torch.int32, device=x.device)
        _check(self.ctx, lib().rot_vote_count_cells(
            self.ctx, _dptr(x, torch.float32, "x"), _dptr(y, torch.float32, "y"), x.shape[0],
            int(B), lins.data_ptr(), m, float(eps), int(mode), a.data_ptr(), b.data_ptr()))
        ca = a.cpu().numpy().view(np.uint32)
        cb = b.cpu().numpy().view(np.uint32)
        return (ca, cb) if mode in (RV_MODE_FINAL, RV_MODE_FINAL_TC) else ca

    def count_cells_culled(self, x, y, B0: int, B: int, lins, eps: float, mode: int,
                           want_bits: bool = False):
        """K3-C test hook: counts of `lins` (resolution B) over their level-0 (B0) ancestors'
        pass lists; (cnt_a[, cnt_b][, bits]) with bits uint32 [m0, ceil(n/256)*8]."""
        import torch
        lins = torch.as_tensor(np.asarray(lins, np.uint32).view(np.int32), device=x.device)
        m, n = lins.numel(), x.shape[0]
        a = torch.zeros(max(m, 1), dtype=torch.int32, device=x.device)
        b = torch.zeros(max(m, 1), dtype=torch.int32, device=x.device)
        bits = None
        if want_bits:
            m0 = lib().rv_grid_candidates(int(B0), None, 0)
            bits = torch.zeros((m0, (n + 255) // 256 * 8), dtype=torch.int32, device=x.device)
        _check(self.ctx, lib().rot_vote_count_cells_culled(
            self.ctx, _dptr(x, torch.float32, "x"), _dptr(y, torch.float32, "y"), n, int(B0),
            int(B), lins.data_ptr() if m else a.data_ptr(), m, float(eps), int(mode),
            a.data_ptr(), b.data_ptr(), bits.data_ptr() if bits is not None else None))
        out = [a.cpu().numpy().view(np.uint32)[:m]]
        if mode == RV_MODE_FINAL:
            out.append(b.cpu().numpy().view(np.uint32)[:m])
        if want_bits:
            out.append(bits.cpu().numpy().view(np.uint32))
        return out[0] if len(out) == 1 else tuple(out)

    def solve_multi(self, x, y, eps: float, K: int, rho: float, levels: int = 0) -> list:
        """NEXT-2: up to K rotations, greedy peaks with suppression angle rho (radians)."""
        import torch
        out = (rv_result * K)()
        nf = C.c_int32()
        _check(self.ctx, lib().rot_vote_solve_multi(
            self.ctx, _dptr(x, torch.float32, "x"), _dptr(y, torch.float32, "y"), x.shape[0],
            float(eps), int(levels), int(K), float(rho), out, C.byref(nf)))
        return [Result.from_c(out[k]) for k in range(nf.value)]

    def rigid(self, x, y, mu_t: float, eps: float, levels: int = 0, t_lo: float = -5.0,
              t_hi: float = 5.0, t_step: float = 0.025, pair_ij=None) -> dict:
        """NEXT-3: rigid pose from point correspondences (pairs + length check -> rotation
        vote -> translation vote).  pair_ij: optional CUDA int32 tensor [cap, 2] receiving the
        kept pairs' (i, j)."""
        import torch
        r = rv_rigid_result()
        pp, cap = None, 0
        if pair_ij is not None:
            pp, cap = _dptr(pair_ij, torch.int32, "pair_ij"), pair_ij.shape[0]
        _check(self.ctx, lib().rot_vote_rigid(
            self.ctx, _dptr(x, torch.float32, "x"), _dptr(y, torch.float32, "y"), x.shape[0],
            float(mu_t), float(eps), int(levels), float(t_lo), float(t_hi), float(t_step),
            C.byref(r), pp, int(cap)))
        return {f: (np.array(getattr(r, f)[:]) if f in ("q", "t", "t_mean") else
                    tuple(getattr(r, f)[:]) if f == "t_cell" else getattr(r, f))
                for f, _ in rv_rigid_result._fields_ if f != "pad_"}

    def translation(self, x, y, q, t_lo: float = -5.0, t_hi: float = 5.0,
                    t_step: float = 0.025):
        """The translation vote alone for rotation q: (lin, votes, bin centre, mean)."""
        import torch
        qq = np.ascontiguousarray(q, np.float64)
        lin, votes = C.c_int64(), C.c_uint32()
        t, tm = np.zeros(3), np.zeros(3)
        _check(self.ctx, lib().rot_vote_translation(
            self.ctx, _dptr(x, torch.float32, "x"), _dptr(y, torch.float32, "y"), x.shape[0],
            qq.ctypes.data, float(t_lo), float(t_hi), float(t_step), C.byref(lin),
            C.byref(votes), t.ctypes.data, tm.ctypes.data))
        return lin.value, votes.value, t, tm

    def alg1(self, x, y, J: int = 180, acc=None):
        """NEXT-4: the paper's Algorithm 1 (J samples per circle, dense B^3 accumulator,
        argmax) on the GPU.  acc: optional CUDA int32 tensor of B^3 entries receiving the
        accumulator.  Returns the rv_alg1_result fields as a dict."""
        import torch
        r = rv_alg1_result()
        ap = _dptr(acc, torch.int32, "acc") if acc is not None else None
        _check(self.ctx, lib().rot_vote_alg1(self.ctx, _dptr(x, torch.float32, "x"),
                                             _dptr(y, torch.float32, "y"), x.shape[0], int(J),
                                             C.byref(r), ap))
        return {"q": np.array(r.q[:]), "votes": r.votes, "cell": tuple(r.cell[:]), "B": r.B,
                "J": r.J, "samples": r.samples, "ms": r.ms, "vote_ms": r.vote_ms,
                "lin": (r.cell[0] * r.B + r.cell[1]) * r.B + r.cell[2]}

    def debug_tc_scores(self, x, y, B: int, lins, eps: float):
        """Raw K3-TC scores S' = s_tc - t (bound threshold), float32 [m, ceil(n/256)*256]."""
        import torch
        lins = torch.as_tensor(np.asarray(lins, np.uint32).view(np.int32), device=x.device)
        m, n = lins.numel(), x.shape[0]
        ld = (n + 255) // 256 * 256
        out = torch.empty((m, ld), dtype=torch.float32, device=x.device)
        _check(self.ctx, lib().rot_vote_debug_tc_scores(
            self.ctx, _dptr(x, torch.float32, "x"), _dptr(y, torch.float32, "y"), n, int(B),
            lins.data_ptr(), m, float(eps), out.data_ptr()))
        return out.cpu().numpy()

    def refine(self, x, y, eps: float, q0, rounds: int = 2, mask=None):
        import torch
        q0 = np.ascontiguousarray(q0, np.float64)
        q = np.zeros(4)
        fl = C.c_int32()
        ni = C.c_uint32()
        mp = _dptr(mask, torch.int32, "mask") if mask is not None else None
        _check(self.ctx, lib().rot_vote_refine(
            self.ctx, _dptr(x, torch.float32, "x"), _dptr(y, torch.float32, "y"), x.shape[0],
            float(eps), q0.ctypes.data, int(rounds), q.ctypes.data, C.byref(fl), C.byref(ni), mp))
        return q, fl.value, ni.value


# ---- host planner (pure C++, usable without a GPU) -----------------------------------------

class Plan:
    """The library's host-side level loop (include/rotvote_plan.h)."""

    def __init__(self, chain, levels: int, n: int, eps: float, guard: float = 1e-5,
                 excl=None, rho: float = 0.0):
        ch = np.ascontiguousarray(chain, np.int32)
        h = C.c_void_p()
        ex = np.ascontiguousarray(excl if excl is not None else np.zeros((0, 4)), np.float64)
        rc = lib().rv_plan_create_ex(ch.ctypes.data, ch.size, int(levels), int(n), float(eps),
                                     float(guard), ex.ctypes.data if ex.size else None,
                                     ex.shape[0], float(rho), C.byref(h))
        if rc != 0:
            raise ValueError("invalid plan arguments")
        self.h = h.value

    def request(self):
        B, mode, m = C.c_int32(), C.c_int32(), C.c_int64()
        ptr = C.POINTER(C.c_uint32)()
        if not lib().rv_plan_request(self.h, C.byref(B), C.byref(mode), C.byref(m), C.byref(ptr)):
            return None
        lins = np.ctypeslib.as_array(ptr, shape=(m.value,)).copy() if m.value else np.zeros(0, np.uint32)
        return B.value, mode.value, lins

    def feed(self, cnt_a, cnt_b=None):
        a = np.ascontiguousarray(cnt_a, np.uint32)
        b = np.ascontiguousarray(cnt_b, np.uint32) if cnt_b is not None else None
        rc = lib().rv_plan_feed(self.h, a.ctypes.data, b.ctypes.data if b is not None else None)
        if rc != 0:
            raise ValueError("plan rejected the counts")

    def result(self) -> rv_plan_result:
        r = rv_plan_result()
        if lib().rv_plan_get_result(self.h, C.byref(r)) != 0:
            raise ValueError("plan not finished")
        return r

    def __del__(self):
        try:
            lib().rv_plan_destroy(self.h)
        except Exception:
            pass


def shard_range(m: int, rank: int, world: int):
    b, e = C.c_int64(), C.c_int64()
    lib().rv_shard_range(int(m), int(rank), int(world), C.byref(b), C.byref(e))
    return b.value, e.value


def cull_groups(B0: int, shape=(1, 2, 2)):
    """(group_of[m0], goff[G+1], gmem[m0]) of the ancestor groups (rotvote_plan.h)."""
    gi, gj, gk = (int(v) for v in shape)
    G = lib().rv_cull_groups(int(B0), gi, gj, gk, None, None, None)
    if G < 0:
        raise ValueError("invalid group shape")
    m0 = lib().rv_grid_candidates(int(B0), None, 0)
    g_of = np.zeros(m0, np.int32)
    goff = np.zeros(G + 1, np.int32)
    gmem = np.zeros(m0, np.int32)
    lib().rv_cull_groups(int(B0), gi, gj, gk, g_of.ctypes.data, goff.ctypes.data, gmem.ctypes.data)
    return g_of, goff, gmem


def cull_partition(B0: int, world: int, shape=(1, 2, 2)):
    """(slice[world+1], gslice[world+1]): level-0 row slices and owned group ranges."""
    gi, gj, gk = (int(v) for v in shape)
    sl = np.zeros(world + 1, np.int64)
    gsl = np.zeros(world + 1, np.int64)
    if lib().rv_cull_partition(int(B0), gi, gj, gk, int(world), sl.ctypes.data, gsl.ctypes.data):
        raise ValueError("invalid partition arguments")
    return sl, gsl


def grid_candidates(B: int) -> np.ndarray:
    m = lib().rv_grid_candidates(int(B), None, 0)
    out = np.zeros(m, np.uint32)
    lib().rv_grid_candidates(int(B), out.ctypes.data, m)
    return out


def unpack_mask(words, n: int) -> np.ndarray:
    """uint32 words (LSB-first) -> bool[n]."""
    w = np.asarray(words).view(np.uint32)
    bits = np.unpackbits(w.view(np.uint8), bitorder="little")
    return bits[:n].astype(bool)
