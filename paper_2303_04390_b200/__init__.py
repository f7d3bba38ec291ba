"""phylograd-b200: O(N) branch-length gradients of the phylogenetic
log-likelihood on B200 (arXiv 2303.04390 hot path).

Thin Python binding of the C ABI in include/phylograd.h: argument
marshalling only.  Every step of an evaluation -- transition matrices (Eq. 1),
post-order pruning (Eq. 2), root likelihood (Eq. 3), pre-order partials
(Eq. 4), the per-edge gradient (Eq. 6-8) and the pattern reduction -- runs in
the CUDA kernels of lib/libphylograd.so.  There is no CPU fallback: if the
native library is missing this module raises at import.

PyTorch supplies device memory (the instance workspace is a torch tensor) and
streams; `torch.distributed` (NCCL) combines pattern shards (see
`allreduce_evaluation`).
"""
from __future__ import annotations

import ctypes
import os
import re
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PHYLOGRAD_LIB", os.path.join(_HERE, "lib", "libphylograd.so"))
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "phylograd.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"native library {LIB_PATH} is missing; build it with "
        "`python paper_2303_04390_b200/build.py` (nvcc, sm_100a). There is no fallback.")

_lib = ctypes.CDLL(LIB_PATH)

# ---- constants (mirrors include/phylograd.h) --------------------------------
PG_OK, PG_ERR_ARG, PG_ERR_DOMAIN, PG_ERR_TOPOLOGY, PG_ERR_SEQUENCE = 0, 1, 2, 3, 4
PG_ERR_ZERO_LIKELIHOOD, PG_ERR_CUDA, PG_ERR_UNSUPPORTED, PG_ERR_MEMORY = 5, 6, 7, 8
PG_FP64, PG_FP32 = 0, 1
PG_FLAG_TIP_PARTIALS = 1


class PgConfig(ctypes.Structure):
    _fields_ = [("tips", ctypes.c_int32), ("patterns", ctypes.c_int32), ("states", ctypes.c_int32),
                ("categories", ctypes.c_int32), ("precision", ctypes.c_int32),
                ("device", ctypes.c_int32), ("flags", ctypes.c_uint32)]


class PgPlanInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("post_depth", "pre_depth", "grid", "block", "smem_bytes",
                                              "prefetch_depth", "padded_patterns", "kernel_variant",
                                              "flow_tiles", "flow_version", "flow_stages", "flow_pdl")]


_vp = ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int32)

_SIGS = {
    "pg_version": ([], ctypes.c_int),
    "pg_workspace_bytes": ([ctypes.POINTER(PgConfig), ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "pg_create": ([ctypes.POINTER(PgConfig), _vp, _vp, ctypes.c_size_t, ctypes.POINTER(_vp)], ctypes.c_int),
    "pg_destroy": ([_vp], ctypes.c_int),
    "pg_set_tip_states": ([_vp, ctypes.c_int32, _ip], ctypes.c_int),
    "pg_set_tip_partials": ([_vp, ctypes.c_int32, _dp], ctypes.c_int),
    "pg_set_pattern_weights": ([_vp, _dp], ctypes.c_int),
    "pg_set_state_frequencies": ([_vp, _dp], ctypes.c_int),
    "pg_set_eigen": ([_vp, _dp, _dp, _dp], ctypes.c_int),
    "pg_set_category_rates": ([_vp, _dp], ctypes.c_int),
    "pg_set_category_weights": ([_vp, _dp], ctypes.c_int),
    "pg_set_operations": ([_vp, _ip, ctypes.c_int32], ctypes.c_int),
    "pg_set_branch_lengths": ([_vp, _dp], ctypes.c_int),
    "pg_set_branch_lengths_device": ([_vp, _vp], ctypes.c_int),
    "pg_set_node_heights": ([_vp, _dp, _dp], ctypes.c_int),
    "pg_set_node_heights_device": ([_vp, _vp, _vp], ctypes.c_int),
    "pg_set_branch_sets": ([_vp, _ip, ctypes.c_int32], ctypes.c_int),
    "pg_clock_gradient_device": ([_vp, _vp, _vp, _vp, _vp], ctypes.c_int),
    "pg_hmc_leapfrog": ([_vp, _vp, _vp, _vp, ctypes.c_double, ctypes.c_int32, _vp, _vp], ctypes.c_int),
    "pg_compute": ([_vp, _dp, _dp], ctypes.c_int),
    "pg_compute_device": ([_vp, _vp], ctypes.c_int),
    "pg_check_status": ([_vp, _ip], ctypes.c_int),
    "pg_kernels_per_eval": ([_vp, _ip], ctypes.c_int),
    "pg_get_plan_info": ([_vp, ctypes.POINTER(PgPlanInfo)], ctypes.c_int),
    "pg_set_kernel_timing": ([_vp, ctypes.c_int], ctypes.c_int),
    "pg_get_kernel_times": ([_vp, ctypes.POINTER(ctypes.c_float)], ctypes.c_int),
    "pg_plan_check": ([ctypes.c_int32, _ip, ctypes.c_int32, _ip, _ip], ctypes.c_int),
    "pg_last_error": ([_vp], ctypes.c_char_p),
    "pg_strerror": ([ctypes.c_int], ctypes.c_char_p),
}
for _name, (_args, _res) in _SIGS.items():
    if not hasattr(_lib, _name):
        raise ImportError(f"{LIB_PATH} lacks {_name} (stale build); rebuild with "
                          "`python paper_2303_04390_b200/build.py`")
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res


def header_symbols() -> list[str]:
    """Every function the C ABI header declares."""
    txt = open(HEADER_PATH).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pg_[a-z_]+)\s*\(", txt)))


class PhyloGradError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_lib.pg_strerror(code).decode()} (code {code}): {msg}")
        self.code = code


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a, n: Optional[int] = None, what: str = "array") -> np.ndarray:
    """C-contiguous float64 copy/view of `a`; with `n`, its size must be n (the
    C side reads exactly that many values: a short array would be a heap
    over-read, a long one a silent truncation)."""
    x = np.ascontiguousarray(a, dtype=np.float64)
    if n is not None and x.size != n:
        raise ValueError(f"{what}: expected {n} values, got {x.size} (shape {np.shape(a)})")
    return x


def _i32(a, n: int, what: str) -> np.ndarray:
    x = np.ascontiguousarray(a, dtype=np.int32)
    if x.size != n:
        raise ValueError(f"{what}: expected {n} values, got {x.size} (shape {np.shape(a)})")
    return x


def plan_check(tips: int, ops) -> tuple[int, int]:
    """Host-only topology validation; returns (post_depth, pre_depth)."""
    o = np.ascontiguousarray(ops, dtype=np.int32).reshape(-1, 3)
    a, b = ctypes.c_int32(0), ctypes.c_int32(0)
    rc = _lib.pg_plan_check(int(tips), o.ctypes.data_as(_ip), int(o.shape[0]), ctypes.byref(a), ctypes.byref(b))
    if rc:
        raise PhyloGradError(rc, "invalid operation list")
    return a.value, b.value


def workspace_bytes(tips, patterns, states, categories, precision="fp64", tip_partials=False) -> int:
    cfg = PgConfig(tips, patterns, states, categories, PG_FP64 if precision == "fp64" else PG_FP32, 0,
                   PG_FLAG_TIP_PARTIALS if tip_partials else 0)
    n = ctypes.c_size_t(0)
    rc = _lib.pg_workspace_bytes(ctypes.byref(cfg), ctypes.byref(n))
    if rc:
        raise PhyloGradError(rc, "pg_workspace_bytes")
    return n.value


class Instance:
    """One likelihood/gradient instance on one GPU (wraps pg_instance*)."""

    def __init__(self, tips: int, patterns: int, states: int, categories: int,
                 precision: str = "fp64", device: int = 0, tip_partials: bool = False,
                 stream=None, torch_workspace: bool = True):
        import torch  # plumbing only: device memory and streams
        self.torch = torch
        self.tips, self.patterns, self.states, self.categories = tips, patterns, states, categories
        self.precision = precision
        self.device = device
        self.cfg = PgConfig(tips, patterns, states, categories,
                            PG_FP64 if precision == "fp64" else PG_FP32, device,
                            PG_FLAG_TIP_PARTIALS if tip_partials else 0)
        nbytes = ctypes.c_size_t(0)
        self._check(_lib.pg_workspace_bytes(ctypes.byref(self.cfg), ctypes.byref(nbytes)), "workspace")
        dev = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.Stream(device=dev)
        self.workspace = (torch.empty(nbytes.value, dtype=torch.uint8, device=dev)
                          if torch_workspace else None)
        self._h = _vp()
        ws_ptr = self.workspace.data_ptr() if self.workspace is not None else None
        ws_len = nbytes.value if self.workspace is not None else 0
        self._check(_lib.pg_create(ctypes.byref(self.cfg), _vp(self.stream.cuda_stream), ws_ptr,
                                   ws_len, ctypes.byref(self._h)), "pg_create")
        self.n_branches = 2 * tips - 2

    # -- plumbing ----------------------------------------------------------
    def _check(self, rc: int, what: str):
        if rc != PG_OK:
            msg = what
            if getattr(self, "_h", None) and self._h.value:
                msg = f"{what}: {_lib.pg_last_error(self._h).decode()}"
            raise PhyloGradError(rc, msg)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.pg_destroy(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- setters (copied at call time; sizes checked here) -------
    def set_tip_states(self, tip: int, states):
        s = _i32(states, self.patterns, "tip states [C]")
        self._check(_lib.pg_set_tip_states(self._h, int(tip), s.ctypes.data_as(_ip)), "set_tip_states")

    def set_tip_partials(self, tip: int, partials):
        p = _f64(partials, self.patterns * self.states, "tip partials [C][S]")
        self._check(_lib.pg_set_tip_partials(self._h, int(tip), _dptr(p)), "set_tip_partials")

    def set_pattern_weights(self, w):
        self._check(_lib.pg_set_pattern_weights(self._h, _dptr(_f64(w, self.patterns, "pattern weights [C]"))),
                    "set_pattern_weights")

    def set_state_frequencies(self, pi):
        self._check(_lib.pg_set_state_frequencies(self._h, _dptr(_f64(pi, self.states, "pi [S]"))),
                    "set_state_frequencies")

    def set_eigen(self, evec, ievec, evals):
        S = self.states
        V, Vi, lam = _f64(evec, S * S, "evec [S][S]"), _f64(ievec, S * S, "ievec [S][S]"), _f64(evals, S, "eval [S]")
        self._check(_lib.pg_set_eigen(self._h, _dptr(V), _dptr(Vi), _dptr(lam)), "set_eigen")

    def set_category_rates(self, rates):
        self._check(_lib.pg_set_category_rates(self._h, _dptr(_f64(rates, self.categories, "category rates [R]"))),
                    "set_category_rates")

    def set_category_weights(self, w):
        self._check(_lib.pg_set_category_weights(self._h, _dptr(_f64(w, self.categories, "category weights [R]"))),
                    "set_category_weights")

    def set_operations(self, ops):
        o = np.ascontiguousarray(ops, dtype=np.int32).reshape(-1, 3)
        self._check(_lib.pg_set_operations(self._h, o.ctypes.data_as(_ip), int(o.shape[0])), "set_operations")

    def set_branch_lengths(self, b):
        self._check(_lib.pg_set_branch_lengths(self._h, _dptr(_f64(b, self.n_branches, "branch lengths [2N-2]"))),
                    "set_branch_lengths")

    def set_branch_lengths_device(self, t):
        """t: a CUDA float64 tensor of 2N-2 branch lengths (stream-ordered copy)."""
        assert t.dtype == self.torch.float64 and t.is_cuda and t.numel() == self.n_branches
        self._check(_lib.pg_set_branch_lengths_device(self._h, _vp(t.data_ptr())), "set_branch_lengths_device")

    # -- time-tree parameterisation (include/phylograd.h) --------
    def set_node_heights(self, heights, rates=None):
        """b_i = rho_i (h_parent(i) - h_i) from host heights [2N-1] and rate
        scalars [2N-2] (None = all 1); validated and copied."""
        r = None if rates is None else _f64(rates, self.n_branches, "rate scalars [2N-2]")
        h = _f64(heights, self.n_branches + 1, "node heights [2N-1]")
        self._check(_lib.pg_set_node_heights(self._h, _dptr(h), _dptr(r) if r is not None else None),
                    "set_node_heights")

    def set_node_heights_device(self, h, rates=None):
        """Same from CUDA float64 tensors (stream-ordered, not validated)."""
        assert h.dtype == self.torch.float64 and h.is_cuda and h.numel() == self.n_branches + 1
        if rates is not None:
            assert rates.dtype == self.torch.float64 and rates.is_cuda and rates.numel() == self.n_branches
        self._check(_lib.pg_set_node_heights_device(self._h, _vp(h.data_ptr()),
                                                    _vp(rates.data_ptr()) if rates is not None else None),
                    "set_node_heights_device")

    def set_branch_sets(self, set_of_branch, n_sets: int):
        s = _i32(set_of_branch, self.n_branches, "branch set ids [2N-2]")
        self._check(_lib.pg_set_branch_sets(self._h, s.ctypes.data_as(_ip), int(n_sets)), "set_branch_sets")

    def clock_gradient_device(self, out, grad_rates=None, grad_heights=None, set_sums=None):
        """Chain rule on the device from out = [logL, g] (compute_device's
        output): dlogL/drho [2N-2], dlogL/dh [2N-1], branch-set sums; any
        output tensor may be None."""
        def ptr(t):
            return None if t is None else _vp(t.data_ptr())
        self._check(_lib.pg_clock_gradient_device(self._h, _vp(out.data_ptr()), ptr(grad_rates),
                                                  ptr(grad_heights), ptr(set_sums)), "clock_gradient_device")

    def clock_gradient(self, n_sets: int = 1):
        """Synchronous evaluation in the time-tree parameterisation: returns
        (logL, g, dlogL/drho, dlogL/dh, set sums) as host arrays."""
        torch = self.torch
        dev = torch.device("cuda", self.device)
        B = self.n_branches
        out = torch.empty(B + 1, dtype=torch.float64, device=dev)
        gr = torch.empty(B, dtype=torch.float64, device=dev)
        gh = torch.empty(B + 1, dtype=torch.float64, device=dev)
        ss = torch.empty(n_sets, dtype=torch.float64, device=dev)
        with torch.cuda.stream(self.stream):
            self.compute_device(out)
            self.clock_gradient_device(out, gr, gh, ss)
        self.stream.synchronize()
        zp = self.check_status()
        if zp >= 0:
            raise PhyloGradError(PG_ERR_ZERO_LIKELIHOOD, f"zero likelihood at pattern {zp}")
        o = out.cpu().numpy()
        return o[0], o[1:], gr.cpu().numpy(), gh.cpu().numpy(), ss.cpu().numpy()

    # -- evaluation ----------------------------------------------------------
    def compute(self, gradient: bool = True):
        """Synchronous evaluation with host outputs: (logL, gradient[2N-2])."""
        logl = ctypes.c_double(0.0)
        g = np.zeros(self.n_branches) if gradient else None
        self._check(_lib.pg_compute(self._h, ctypes.byref(logl), _dptr(g) if g is not None else None),
                    "compute")
        return logl.value, g

    def compute_device(self, out):
        """Asynchronous evaluation into a CUDA float64 tensor out[2N-1] =
        [logL, g_0..g_{2N-3}] (this instance's partial sums), on self.stream."""
        assert out.dtype == self.torch.float64 and out.is_cuda and out.numel() >= self.n_branches + 1
        self._check(_lib.pg_compute_device(self._h, _vp(out.data_ptr())), "compute_device")

    def hmc_leapfrog(self, theta, p, eps: float, n_steps: int, out, inv_mass=None, grad_theta=None):
        """n_steps leapfrog steps over theta = log b on the device (NEXT-4,
        include/phylograd.h pg_hmc_leapfrog): theta, p (float64 CUDA tensors,
        [2N-2]) are updated in place; out [2N-1] receives [logL, dlogL/db] and
        grad_theta (optional) the gradient of logL + sum(theta) at the end."""
        t = self.torch
        for x in (theta, p, out) + tuple(y for y in (inv_mass, grad_theta) if y is not None):
            assert x.dtype == t.float64 and x.is_cuda and x.is_contiguous()

        def ptr(x):
            return None if x is None else _vp(x.data_ptr())
        self._check(_lib.pg_hmc_leapfrog(self._h, ptr(theta), ptr(p), ptr(inv_mass), float(eps), int(n_steps),
                                         ptr(out), ptr(grad_theta)), "hmc_leapfrog")

    def check_status(self) -> int:
        zp = ctypes.c_int32(-1)
        rc = _lib.pg_check_status(self._h, ctypes.byref(zp))
        if rc not in (PG_OK, PG_ERR_ZERO_LIKELIHOOD):
            self._check(rc, "check_status")
        return zp.value

    def set_kernel_timing(self, enable: bool = True):
        self._check(_lib.pg_set_kernel_timing(self._h, int(enable)), "set_kernel_timing")

    def kernel_times(self) -> dict:
        """Device milliseconds of each kernel of the most recent evaluation."""
        ms = (ctypes.c_float * 3)()
        self._check(_lib.pg_get_kernel_times(self._h, ms), "get_kernel_times")
        return {"pmat": ms[0], "traverse": ms[1], "reduce": ms[2]}

    def kernels_per_eval(self) -> int:
        n = ctypes.c_int32(0)
        self._check(_lib.pg_kernels_per_eval(self._h, ctypes.byref(n)), "kernels_per_eval")
        return n.value

    def plan_info(self) -> dict:
        info = PgPlanInfo()
        self._check(_lib.pg_get_plan_info(self._h, ctypes.byref(info)), "plan_info")
        return {f: getattr(info, f) for f, _ in PgPlanInfo._fields_}


def from_problem(pb, precision: Optional[str] = None, device: int = 0, stream=None,
                 lo: int = 0, hi: Optional[int] = None) -> Instance:
    """Instance loaded with a phylo_synth.Problem (optionally a pattern shard)."""
    hi = pb.patterns if hi is None else hi
    C = hi - lo
    part = pb.has_partials
    inst = Instance(pb.n_tips, C, pb.states, len(pb.cat_rates),
                    precision=precision or pb.precision, device=device, tip_partials=part, stream=stream)
    for n in range(pb.n_tips):
        if part:
            inst.set_tip_partials(n, pb.tip_partial_rows(n, lo, hi))
        else:
            inst.set_tip_states(n, pb.tip_states[n, lo:hi])
    inst.set_pattern_weights(pb.pattern_weights[lo:hi])
    inst.set_state_frequencies(pb.pi)
    inst.set_eigen(pb.evec, pb.ievec, pb.evals)
    inst.set_category_rates(pb.cat_rates)
    inst.set_category_weights(pb.cat_weights)
    inst.set_operations(pb.ops)
    inst.set_branch_lengths(pb.branch_lengths)
    return inst


def shard_range(C: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous pattern shard [lo, hi) of `rank`: patterns
    are conditionally independent, so logL and every gradient
    entry are sums of per-shard partial sums (Eq. 6).  Balanced
    split: shard sizes differ by at most one; a shard is empty only when
    C < world (then that rank contributes zeros to the allreduce)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return rank * C // world, (rank + 1) * C // world


def allreduce_evaluation(out, group=None):
    """A7: sum the per-shard [logL, g] vector across ranks (one allreduce per
    evaluation, on the current stream; NCCL on GPUs).  It may be captured in
    the same CUDA graph as pg_compute_device (see `capture_evaluation`)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():      # world size 1 too: the same collective path
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out


class ShardEvaluation:
    """One rank's side of a pattern-sharded evaluation.

    `pb` is a phylo_synth.Problem (the whole alignment); this rank evaluates
    patterns shard_range(C, world, rank) through the C ABI and the per-shard
    [logL, g] vectors are summed with one allreduce.  A rank whose shard is
    empty (C < world) creates no instance and contributes zeros.

    capture=True records [set_branch_lengths_device, compute_device,
    allreduce] as ONE CUDA graph on the instance stream (the library enqueues
    into the caller's capture) and replays it per evaluation.
    """

    def __init__(self, pb, rank: int = 0, world: int = 1, device: int = 0, precision: Optional[str] = None,
                 group=None, capture: bool = False, timing: bool = False):
        import torch
        self.torch = torch
        self.group = group
        self.lo, self.hi = shard_range(pb.patterns, world, rank)
        self.n_branches = 2 * pb.n_tips - 2
        self.dev = torch.device("cuda", device)
        self.inst = from_problem(pb, precision=precision, device=device, lo=self.lo, hi=self.hi) \
            if self.hi > self.lo else None
        self.stream = self.inst.stream if self.inst is not None else torch.cuda.Stream(device=self.dev)
        self.out = torch.zeros(self.n_branches + 1, dtype=torch.float64, device=self.dev)
        self.bl = torch.tensor(np.asarray(pb.branch_lengths[:self.n_branches], dtype=np.float64), device=self.dev)
        self.graph = None
        if timing and self.inst is not None:          # per-kernel events (recorded inside the graph too)
            self.inst.set_kernel_timing(True)
        if capture:
            with torch.cuda.stream(self.stream):
                self._enqueue()                       # uploads + plan outside the capture
            self.stream.synchronize()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=self.stream):
                self._enqueue()

    def _enqueue(self):
        if self.inst is not None:
            self.inst.set_branch_lengths_device(self.bl)
            self.inst.compute_device(self.out)
        else:
            self.out.zero_()
        allreduce_evaluation(self.out, self.group)

    def evaluate(self, branch_lengths=None):
        """[logL, g] summed over all ranks' shards (device tensor, stream-ordered)."""
        torch = self.torch
        with torch.cuda.stream(self.stream):
            if branch_lengths is not None:
                self.bl.copy_(torch.as_tensor(np.asarray(branch_lengths, dtype=np.float64)), non_blocking=False)
            if self.graph is not None:
                self.graph.replay()
            else:
                self._enqueue()
        return self.out

    def zero_pattern(self) -> int:
        """First zero-likelihood pattern of this shard (global index) or -1."""
        if self.inst is None:
            return -1
        zp = self.inst.check_status()
        return zp + self.lo if zp >= 0 else -1

    def close(self):
        if self.inst is not None:
            self.inst.close()
            self.inst = None
