"""Device residency of an instance: torch CUDA buffers + a libpdcs engine.

PyTorch is used only to allocate device memory and to own the CUDA stream;
all arithmetic runs in libpdcs kernels (include/pdcs.h).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import _native as N
from .model import KIND_CODE, ConicProblem, dual_layout


def _torch():
    import torch

    return torch


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def _dev_f64(arr, stream=None):
    torch = _torch()
    a = np.ascontiguousarray(arr, dtype=np.float64)
    t = torch.empty(max(a.size, 1), dtype=torch.float64, device="cuda")
    if a.size:
        t[: a.size].copy_(torch.from_numpy(a), non_blocking=False)
    return t


def _dev_i32(arr):
    torch = _torch()
    a = np.ascontiguousarray(arr, dtype=np.int32)
    t = torch.empty(max(a.size, 1), dtype=torch.int32, device="cuda")
    if a.size:
        t[: a.size].copy_(torch.from_numpy(a))
    return t


def _empty_f64(n):
    torch = _torch()
    return torch.zeros(max(int(n), 1), dtype=torch.float64, device="cuda")


def _slab(dtype, sizes: dict, align: int = 64) -> dict:
    """Zeroed device views carved out of ONE allocation: a fresh cudaMalloc per
    large buffer costs ~14 ms on the B200 box (tools/xfer_probe.py: 33
    vectors 0.47 s, one 4 GB slab 5 ms), which dominated engine setup."""
    torch = _torch()
    offs, total = {}, 0
    for name, count in sizes.items():
        offs[name] = total
        total += -(-max(int(count), 1) // align) * align
    buf = torch.zeros(max(total, 1), dtype=dtype, device="cuda")
    return {name: buf[off:off + max(int(sizes[name]), 1)] for name, off in offs.items()}


_STAGE_BYTES = int(os.environ.get("PDCS_STAGE_MB", "32")) << 20
_NSTAGE = max(2, int(os.environ.get("PDCS_STAGES", "2")))  # pinned buffers per thread (upload pipeline depth)
_stage_local = threading.local()
# set by batch.solve_many's thread-pool path: engines built on this thread stay
# on the CUDA-graph path (a persistent cooperative launch occupies the GPU)
_thread_opts = threading.local()
# host threads of the large staged copies (PDCS_COPY_THREADS overrides): copies
# into freshly allocated result arrays are page-fault bound (one thread: 5 GB/s,
# four: 18 GB/s; tools/host_copy_probe.py); 8 took C5's download 36-40 -> 30-34 ms
_COPY_THREADS = max(1, int(os.environ.get("PDCS_COPY_THREADS", str(min(8, os.cpu_count() or 4)))))
_copy_pool = None
_copy_lock = threading.Lock()


def _pcopy(dst: np.ndarray, src: np.ndarray) -> None:
    """dst[:] = src (flat uint8 views) with up to _COPY_THREADS host threads (numpy
    releases the GIL in the copy): ~19 GB/s into pinned memory instead of
    ~8.5 on one thread, the host side of every large upload / download."""
    global _copy_pool
    n = src.size
    if n < (4 << 20):
        dst[:] = src
        return
    with _copy_lock:
        if _copy_pool is None:
            from concurrent.futures import ThreadPoolExecutor

            _copy_pool = ThreadPoolExecutor(max_workers=_COPY_THREADS, thread_name_prefix="pdcs-copy")
    k = _COPY_THREADS
    cuts = [n * i // k for i in range(k + 1)]

    def part(i):
        dst[cuts[i]:cuts[i + 1]] = src[cuts[i]:cuts[i + 1]]

    list(_copy_pool.map(part, range(k)))


def _stages():
    """Two reusable pinned host buffers for double-buffered transfers, one
    pair per host thread: `solve_many` runs concurrent solves on several
    threads, and a shared pair would let one thread overwrite a chunk another
    thread's async copy is still reading."""
    bufs = getattr(_stage_local, "bufs", None)
    if bufs is None:
        torch = _torch()
        bufs = [torch.empty(_STAGE_BYTES, dtype=torch.uint8, pin_memory=True) for _ in range(_NSTAGE)]
        _stage_local.bufs = bufs
    return bufs


def h2d(dst, arr, stream) -> None:
    """Host array -> device view `dst` (same dtype) through double-buffered
    pinned staging on `stream` (~30 GB/s; a pageable copy runs at ~10)."""
    torch = _torch()
    np_dtype = {torch.float64: np.float64, torch.int32: np.int32}[dst.dtype]
    a = np.ascontiguousarray(arr, dtype=np_dtype).reshape(-1)
    if a.size == 0:
        return
    if a.nbytes < (1 << 20):
        with torch.cuda.stream(stream):
            dst[: a.size].copy_(torch.from_numpy(a), non_blocking=False)
        stream.synchronize()
        return
    src = a.view(np.uint8)
    dbytes = dst[: a.size].view(torch.uint8)
    st = _stages()
    done = [None] * len(st)
    with torch.cuda.stream(stream):
        for i, off in enumerate(range(0, src.size, _STAGE_BYTES)):
            b = i % len(st)
            if done[b] is not None:
                done[b].synchronize()
            k = min(_STAGE_BYTES, src.size - off)
            _pcopy(st[b][:k].numpy(), src[off:off + k])
            dbytes[off:off + k].copy_(st[b][:k], non_blocking=True)
            done[b] = torch.cuda.Event()
            done[b].record(stream)
    stream.synchronize()


def d2h(src, n: int, stream) -> np.ndarray:
    """First n elements of a device tensor -> new host array, through the
    pinned staging buffers (the next chunk's DMA overlaps this chunk's copy)."""
    torch = _torch()
    np_dtype = {torch.float64: np.float64, torch.int32: np.int32}[src.dtype]
    out = np.empty(n, dtype=np_dtype)
    if n == 0:
        return out
    if out.nbytes < (1 << 20):
        with torch.cuda.stream(stream):
            host = src[:n].cpu()
        return host.numpy().copy()
    ob = out.view(np.uint8)
    sb = src[:n].view(torch.uint8)
    st = _stages()
    chunks = list(range(0, ob.size, _STAGE_BYTES))
    events = []
    with torch.cuda.stream(stream):
        def issue(i):
            off = chunks[i]
            k = min(_STAGE_BYTES, ob.size - off)
            st[i & 1][:k].copy_(sb[off:off + k], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            events.append(ev)

        issue(0)
        for i, off in enumerate(chunks):
            if i + 1 < len(chunks):
                issue(i + 1)
            events[i].synchronize()
            k = min(_STAGE_BYTES, ob.size - off)
            _pcopy(ob[off:off + k], st[i & 1][:k].numpy())
    return out


class DeviceCSR:
    """Device copy of a CSR matrix and of its (device-built) transpose, for
    SparseMatrix.matvec / rmatvec."""

    def __init__(self, csr):
        lib = N.lib()
        torch = _torch()
        self.m, self.n = csr.shape
        self.nnz = int(csr.nnz)
        self.rp = _dev_i32(csr.indptr)
        self.ci = _dev_i32(csr.indices)
        self.va = _dev_f64(csr.data)
        self.trp = torch.zeros(self.n + 1, dtype=torch.int32, device="cuda")
        self.tci = torch.empty(max(self.nnz, 1), dtype=torch.int32, device="cuda")
        self.tva = torch.empty(max(self.nnz, 1), dtype=torch.float64, device="cuda")
        self.perm = torch.empty(max(self.nnz, 1), dtype=torch.int32, device="cuda")
        torch.cuda.current_stream().synchronize()
        N.check(lib.pdcs_transpose_csr(self.m, self.n, self.nnz, _ptr(self.rp), _ptr(self.ci),
                                       _ptr(self.va), _ptr(self.trp), _ptr(self.tci),
                                       _ptr(self.tva), _ptr(self.perm), None), "pdcs_transpose_csr")

    def _apply(self, rows, rp, ci, va, v):
        lib = N.lib()
        x = _dev_f64(v)
        y = _empty_f64(rows)
        N.check(lib.pdcs_spmv_csr(rows, _ptr(rp), _ptr(ci), _ptr(va), _ptr(x), _ptr(y), None),
                "pdcs_spmv_csr")
        return y[:rows].cpu().numpy()

    def matvec(self, x):
        if self.m == 0:
            return np.zeros(0)
        return self._apply(self.m, self.rp, self.ci, self.va, x)

    def rmatvec(self, y):
        if self.n == 0:
            return np.zeros(0)
        return self._apply(self.n, self.trp, self.tci, self.tva, y)


def project_segments(v: np.ndarray, blocks, scale: np.ndarray | None = None,
                     root_tol: float = 1e-12, max_root_iters: int = 100) -> np.ndarray:
    """Segmented cone projection of a host vector on the GPU.

    blocks: iterable of (kind_code, start, dim, smode); root_tol /
    max_root_iters: the ProjectionSettings fields.  Returns (out, err)."""
    lib = N.lib()
    v = np.ascontiguousarray(v, dtype=np.float64)
    blocks = list(blocks)
    arr = (N.PdcsBlock * max(len(blocks), 1))()
    for i, (k, s, d, sm) in enumerate(blocks):
        arr[i] = N.PdcsBlock(int(k), int(s), int(d), int(sm))
    din = _dev_f64(v)
    dout = _empty_f64(v.size)
    dsc = _dev_f64(scale) if scale is not None else None
    err = C.c_int32(0)
    N.check(lib.pdcs_project_segments_ex(v.size, _ptr(din), _ptr(dout), arr, len(blocks), _ptr(dsc),
                                         float(root_tol), int(max_root_iters), C.byref(err), None),
            "pdcs_project_segments_ex")
    return dout[: v.size].cpu().numpy(), int(err.value)


def project_box_dev(v, l, u):
    lib = N.lib()
    v = np.ascontiguousarray(v, dtype=np.float64)
    dv, dl, du = _dev_f64(v), _dev_f64(l), _dev_f64(u)
    out = _empty_f64(v.size)
    N.check(lib.pdcs_project_box(v.size, _ptr(dv), _ptr(dl), _ptr(du), _ptr(out), None),
            "pdcs_project_box")
    return out[: v.size].cpu().numpy()


def axpby_dev(a, p, b, q, d=1.0):
    """(a p + b q) / d on the GPU for host vectors (q may be None)."""
    lib = N.lib()
    p = np.ascontiguousarray(p, dtype=np.float64)
    dp = _dev_f64(p)
    dq = _dev_f64(q) if q is not None else None
    out = _empty_f64(p.size)
    N.check(lib.pdcs_vec_axpby(p.size, float(a), _ptr(dp), float(b), _ptr(dq), float(d), _ptr(out), None),
            "pdcs_vec_axpby")
    return out[: p.size].cpu().numpy()


class DeviceEngine:
    """A presolved (post-RSOC) instance resident on the GPU with all solver
    state buffers and a libpdcs engine handle.

    mode "scale": Ruiz/PC preconditioning on the device (or identity when
    use_preconditioner is off); mode "asis": the instance is used exactly as
    given, with its ConeSpec scales as the block scales (step-level API)."""

    def __init__(self, work: ConicProblem, *, asis: bool = False, allow_nonuniform_dual_soc=False,
                 x_pad: int = 0):
        """x_pad: extra elements on the x-space iterate buffers (a sharded
        engine's NCCL all-gather / reduce-scatter of x-slices needs
        nranks * ceil(n / nranks) of them)."""
        lib = N.lib()
        torch = _torch()
        self.lib = lib
        self.work = work
        self.stream = torch.cuda.Stream()
        n, m = work.n, work.m
        self.n, self.m, self.nbox = n, m, work.num_box
        csr = work.G._csr
        self.nnz = int(csr.nnz)
        self.m_zero, self.m_elem = dual_layout(work)
        nb, nnz = work.num_box, self.nnz
        names_x = ["x", "xh", "xb", "xa", "xpa", "gty", "gtya", "gth", "gtr", "xt",
                   "tx0", "tx1", "tx2", "px0", "px1", "px2", "pgty"]
        names_y = ["y", "yh", "yb", "ya", "ypa", "gx", "gxa", "w", "gxh",
                   "ty0", "ty1", "ty2", "py0", "py1", "py2", "pgx"]
        f64 = {"g_val0": nnz, "g_val": nnz, "gt_val": nnz, "c0": n, "h0": m, "l0": nb, "u0": nb,
               "c": n, "h": m, "l": nb, "u": nb, "d1": m, "d2": n}
        f64.update({nm: n + x_pad for nm in names_x})
        f64.update({nm: m for nm in names_y})
        i32 = {"g_rowptr": m + 1, "g_colidx": nnz, "gt_rowptr": n + 1, "gt_colidx": nnz, "perm": nnz}
        with torch.cuda.stream(self.stream):
            for name, view in {**_slab(torch.float64, f64), **_slab(torch.int32, i32)}.items():
                setattr(self, name, view)
        # stream-level syncs only: a device-wide sync is illegal while another
        # thread's engine captures its graph (concurrent solves, batch.py)
        self.stream.synchronize()
        h2d(self.g_rowptr, csr.indptr, self.stream)
        h2d(self.g_colidx, csr.indices, self.stream)
        h2d(self.g_val0, csr.data, self.stream)
        h2d(self.c0, work.c, self.stream)
        h2d(self.h0, work.h, self.stream)
        h2d(self.l0, work.l, self.stream)
        h2d(self.u0, work.u, self.stream)
        if asis:
            d2 = np.ones(n)
            for spec, sl in _slices(work.primal_cones, work.num_box):
                d2[sl] = spec.scale
            d1 = np.ones(m)
            for spec, sl in _slices(work.dual_cones, 0):
                d1[sl] = spec.scale
            h2d(self.d1, d1, self.stream)
            h2d(self.d2, d2, self.stream)
        self.stream.synchronize()

        pk = [KIND_CODE[s.kind] for s in work.primal_cones]
        pd = [s.dim for s in work.primal_cones]
        dk = [KIND_CODE[s.kind] for s in work.dual_cones]
        dd = [s.dim for s in work.dual_cones]
        self._keep = [(C.c_int32 * max(len(a), 1))(*a) for a in (pk, pd, dk, dd)]
        desc = N.PdcsEngineDesc()
        desc.n, desc.m, desc.num_box, desc.nnz = n, m, work.num_box, self.nnz
        desc.m_zero, desc.m_elem = self.m_zero, self.m_elem
        desc.n_pcones, desc.n_dcones = len(pk), len(dk)
        desc.h_pcone_kind, desc.h_pcone_dim, desc.h_dcone_kind, desc.h_dcone_dim = self._keep
        desc.allow_nonuniform_dual_soc = int(bool(allow_nonuniform_dual_soc))
        for p in N._DESC_PTRS:
            setattr(desc, p, _ptr(getattr(self, p[2:])))
        self.desc = desc
        h = C.c_void_p()
        N.check(lib.pdcs_engine_create(C.byref(desc), C.c_void_p(self.stream.cuda_stream), C.byref(h)),
                "pdcs_engine_create")
        self.handle = h
        self.asis = asis
        if getattr(_thread_opts, "no_persist", False):
            N.check(lib.pdcs_engine_set_persist(h, 0), "pdcs_engine_set_persist")
        nb = work.num_box
        if nb > 0:
            # uniform box bounds, tested on the uploaded copies (a host np.all over
            # C5's two 160 MB bound vectors cost ~60 ms of the end-to-end solve)
            with torch.cuda.stream(self.stream):
                lv, uv = self.l0[:nb], self.u0[:nb]
                ends = torch.stack([lv[0], uv[0], ((lv == lv[0]).all() & (uv == uv[0]).all()).to(lv.dtype)])
                lo, hi, uni = ends.tolist()
            if uni == 1.0:
                N.check(lib.pdcs_engine_set_uniform_box(h, float(lo), float(hi)), "pdcs_engine_set_uniform_box")

    def close(self):
        """Destroy the libpdcs engine now (solve() calls this when it returns:
        left to the garbage collector, the destroy -- pool frees and a stream
        sync -- could land in the middle of the next solve's setup)."""
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self.lib.pdcs_engine_destroy(h)
            except Exception:  # noqa: BLE001 - interpreter shutdown
                pass
            self.handle = None

    def __del__(self):
        self.close()

    # -- thin wrappers ------------------------------------------------------
    def precondition(self, enabled: int, ruiz_iters: int = 10, use_pc: bool = True):
        N.check(self.lib.pdcs_precondition(self.handle, int(enabled), int(ruiz_iters), int(bool(use_pc))),
                "pdcs_precondition")

    def stats(self):
        out = (C.c_double * 8)()
        N.check(self.lib.pdcs_stats(self.handle, out), "pdcs_stats")
        return dict(c1=out[0], h1=out[1], c2=out[2], h2=out[3], gmax=out[4], rowsum_max=out[5])

    def info(self) -> dict:
        out = (C.c_double * 16)()
        N.check(self.lib.pdcs_engine_info(self.handle, out), "pdcs_engine_info")
        keys = ["vw_g", "vw_gt", "grid_step_x", "grid_step_y", "grid_step_t", "keep_xt", "keep_yh",
                "l2_persist_bytes", "long_rows_g", "long_rows_gt", "primal_blocks", "dual_blocks",
                "panels_g", "panels_gt", "step_vw_g", "step_vw_gt"]
        return {k: out[i] for i, k in enumerate(keys)}

    def get_ctrl(self) -> N.PdcsCtrl:
        c = N.PdcsCtrl()
        N.check(self.lib.pdcs_engine_get_ctrl(self.handle, C.byref(c)), "pdcs_engine_get_ctrl")
        return c

    def set_ctrl(self, c: N.PdcsCtrl):
        N.check(self.lib.pdcs_engine_set_ctrl(self.handle, C.byref(c)), "pdcs_engine_set_ctrl")

    def run_inner(self, slots: int):
        N.check(self.lib.pdcs_run_inner(self.handle, int(slots)), "pdcs_run_inner")

    def profile_slot(self, reps: int):
        """Per-stage device times (ms) of `reps` eager line-search trials."""
        ms = (C.c_double * 32)()
        names = (C.c_char_p * 32)()
        k = self.lib.pdcs_profile_slot(self.handle, int(reps), ms, names, 32)
        if k < 0 or k > 32:
            N.check(1, "pdcs_profile_slot")
        if k == 1 and names[0] is None:
            N.check(1, "pdcs_profile_slot")
        return [(names[i].decode(), ms[i]) for i in range(k)]

    def flush(self):
        N.check(self.lib.pdcs_flush(self.handle), "pdcs_flush")

    def spmv(self, transpose: bool, src, dst):
        N.check(self.lib.pdcs_engine_spmv(self.handle, int(transpose), _ptr(src), _ptr(dst)),
                "pdcs_engine_spmv")

    def metrics(self, mode: int, x, y, gx, gty) -> np.ndarray:
        out = (C.c_double * N.NMET)()
        rc = self.lib.pdcs_metrics(self.handle, int(mode), _ptr(x), _ptr(y), _ptr(gx), _ptr(gty), out)
        if rc == 3:
            from .linalg import NumericalError

            raise NumericalError(self.lib.pdcs_last_error().decode())
        N.check(rc, "pdcs_metrics")
        return np.array(out[:], dtype=np.float64)

    def rays(self, x, y, gx, gty, xnorm, ynorm) -> np.ndarray:
        out = (C.c_double * N.NRAY)()
        rc = self.lib.pdcs_rays(self.handle, _ptr(x), _ptr(y), _ptr(gx), _ptr(gty), float(xnorm),
                                float(ynorm), out)
        if rc == 3:
            from .linalg import NumericalError

            raise NumericalError(self.lib.pdcs_last_error().decode())
        N.check(rc, "pdcs_rays")
        return np.array(out[:], dtype=np.float64)

    def gap_probe(self, x, y, gx, gty, t, tau, sigma):
        out = (C.c_double * 4)()
        rc = self.lib.pdcs_gap_probe(self.handle, _ptr(x), _ptr(y), _ptr(gx), _ptr(gty), float(t),
                                     float(tau), float(sigma), out)
        if rc == 3:
            from .linalg import NumericalError

            raise NumericalError(self.lib.pdcs_last_error().decode())
        N.check(rc, "pdcs_gap_probe")
        return out[0], out[1], out[2], out[3]

    GAP_BATCH = 16  # probes per pdcs_gap_probes call

    def gap_probes(self, x, y, gx, gty, ts, tau, sigma):
        """pdcs_gap_probes: [(dx2, dy2, b1dx, b2dy)] for each t in ts (<= 16)."""
        k = len(ts)
        tsa = (C.c_double * k)(*[float(t) for t in ts])
        out = (C.c_double * (4 * k))()
        rc = self.lib.pdcs_gap_probes(self.handle, _ptr(x), _ptr(y), _ptr(gx), _ptr(gty), tsa, k,
                                      float(tau), float(sigma), out)
        if rc == 3:
            from .linalg import NumericalError

            raise NumericalError(self.lib.pdcs_last_error().decode())
        N.check(rc, "pdcs_gap_probes")
        return [tuple(out[4 * i:4 * i + 4]) for i in range(k)]

    def dist2(self, space: int, a, b=None) -> float:
        out = (C.c_double * 1)()
        N.check(self.lib.pdcs_dist2(self.handle, int(space), _ptr(a), _ptr(b), out), "pdcs_dist2")
        return float(out[0])

    def dot_diff(self, space: int, a, b, c, d) -> float:
        out = (C.c_double * 1)()
        N.check(self.lib.pdcs_dot_diff(self.handle, int(space), _ptr(a), _ptr(b), _ptr(c), _ptr(d), out),
                "pdcs_dot_diff")
        return float(out[0])

    def project_set(self, which: int, src, dst, root_tol: float = 1e-12, max_root_iters: int = 100):
        rc = self.lib.pdcs_project_set_ex(self.handle, int(which), _ptr(src), _ptr(dst), float(root_tol),
                                          int(max_root_iters))
        if rc == 3:
            from .linalg import NumericalError

            raise NumericalError(self.lib.pdcs_last_error().decode())
        N.check(rc, "pdcs_project_set")

    def step_input(self, space: int, v, g, step: float, out):
        N.check(self.lib.pdcs_step_input(self.handle, int(space), _ptr(v), _ptr(g), float(step), _ptr(out)),
                "pdcs_step_input")

    def axpby(self, space: int, a: float, p, b: float, q, out):
        N.check(self.lib.pdcs_axpby(self.handle, int(space), float(a), _ptr(p), float(b), _ptr(q), _ptr(out)),
                "pdcs_axpby")

    def unscale(self, x, y, gx, gty, xo, yo, slack, lam):
        N.check(self.lib.pdcs_unscale(self.handle, _ptr(x), _ptr(y), _ptr(gx), _ptr(gty), _ptr(xo),
                                      _ptr(yo), _ptr(slack), _ptr(lam)), "pdcs_unscale")

    def inject_nan(self, after: int):
        N.check(self.lib.pdcs_debug_inject_nan(self.handle, int(after)), "pdcs_debug_inject_nan")

    # -- buffer helpers -------------------------------------------------------
    def copy(self, dst, src):
        with _torch().cuda.stream(self.stream):
            dst.copy_(src)

    def zero(self, *bufs):
        with _torch().cuda.stream(self.stream):
            for b in bufs:
                b.zero_()

    def upload(self, dst, arr):
        h2d(dst, arr, self.stream)

    def host(self, t, n) -> np.ndarray:
        return d2h(t, n, self.stream)

    def xh_host(self, name):
        return self.host(getattr(self, name), self.n)

    def yh_host(self, name):
        return self.host(getattr(self, name), self.m)


_ENGINES: dict = {}


def engine_for(problem: ConicProblem, original_mode: bool = False) -> DeviceEngine:
    """Cached device engine of an instance for the step-level API.

    original_mode=False: the instance as given, its ConeSpec scales acting as
    block scales (what the reference's project_* / compute_errors see).
    original_mode=True: unit block scales (the unscaled work instance the
    termination checks run on)."""
    import weakref

    if problem.has_rsoc_blocks():
        raise ValueError("rotated blocks must be reformulated (rsoc_to_soc) before projection")
    key = (id(problem), bool(original_mode))
    hit = _ENGINES.get(key)
    if hit is not None and hit[0]() is problem:
        return hit[1]
    e = DeviceEngine(problem, asis=not original_mode)
    e.precondition(0 if original_mode else 2)
    _ENGINES[key] = (weakref.ref(problem, lambda _r, k=key: _ENGINES.pop(k, None)), e)
    return e


def _slices(specs, offset):
    out, start = [], offset
    for s in specs:
        out.append((s, slice(start, start + s.dim)))
        start += s.dim
    return out
