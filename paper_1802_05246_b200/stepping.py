"""Half-step advance of the dissipative and conservative Hermite schemes.

Drop-in replacements for
  hermwave.dissipative.half_step_1d / half_step_2d   (dissipative.py:160-181, 215-247)
  hermwave.conservative.full_step_conservative        (conservative.py:139-157)
  hermwave.conservative.bootstrap_first_half          (conservative.py:166-195)
with the same signatures, validation, parity flip and time bookkeeping.  The
arithmetic runs in one fused sm_100a kernel per call (2D: the cell-map kernel
of csrc/cellmap.cuh; 1D: csrc/line1d.cuh) behind the C ABI of include/hermb200.h.

``advance_*`` run many half steps on device-resident state with two
ping-pong buffers (the throughput path used by bench.py).
"""

from __future__ import annotations

import ctypes as C
import warnings

import numpy as np

from . import _lib as L
from .config import BoundarySpec, BoundarySpec2D, SchemeConfig, check_periodicity
from .device import Staging, ptr, require_cuda, stream_handle
from .fields import DUAL, PRIMAL, Field1D, Field2D, FieldPair, TwoLevelState, flip

_PARITY = {PRIMAL: L.HW_PRIMAL, DUAL: L.HW_DUAL}


def rows2d(t, nrows=None, row0=0, halo_lo=None, halo_hi=None) -> L.Rows2D:
    n = int(t.shape[0]) if nrows is None else int(nrows)
    return L.Rows2D(ptr(t), ptr(halo_lo) if halo_lo is not None else None,
                    ptr(halo_hi) if halo_hi is not None else None, int(row0), n)


def geom2d(grid, parity: str, bc: BoundarySpec2D, trow0: int = 0, ntrows: int = -1) -> L.Geom2D:
    for spec in (bc.x, bc.y):
        check_periodicity(spec, grid.periodic)
    return L.Geom2D(grid.axis(0).n_nodes(parity), grid.axis(1).n_nodes(parity), _PARITY[parity],
                    int(bool(grid.periodic)), L.axis_bc(bc.x), L.axis_bc(bc.y), int(trow0), int(ntrows))


def _target_shape2d(grid, parity_src: str, kx: int, ky: int):
    tp = flip(parity_src)
    return (grid.axis(0).n_nodes(tp), grid.axis(1).n_nodes(tp), kx + 1, ky + 1)


def _min_h(field) -> float:
    if isinstance(field, Field1D):
        return field.grid.h
    return min(field.grid.hx, field.grid.hy)


# ---------------------------------------------------------------- 2D dissipative

def diss2d_into(u, v, ud, vd, grid, parity, m, cfg: SchemeConfig, bc: BoundarySpec2D, stream=None):
    """Raw device call: u/v (source parity) -> ud/vd (flipped parity)."""
    dt = cfg.dt(min(grid.hx, grid.hy))
    g = geom2d(grid, parity, bc)
    cap = -1 if cfg.stage_cap is None else int(cfg.stage_cap)
    s = stream if stream is not None else stream_handle(u.device)
    L.check(L.lib().hw_diss2d_half_step(C.byref(rows2d(u)), C.byref(rows2d(v)), ptr(ud), ptr(vd), int(m),
                                        C.byref(g), dt, grid.hx, grid.hy, cfg.speed, cap, s),
            "half_step_2d")
    return dt


def _diss2d_host_pipelined(uh, vh, grid, parity, m, cfg: SchemeConfig, bc: BoundarySpec2D, nchunks: int = 16,
                           _marks=None, _interleave=None, _pinned=None):
    """Host arrays in, host arrays out, with the PCIe traffic overlapped: the
    source rows go up in chunks on one stream, each target-row chunk launches
    as soon as the source rows it reads (its flanking rows, periodic wrap or
    wall mirror included) have landed, and its results come back on a third
    stream while the next chunk computes.  Same arithmetic as the one-shot
    path (the kernel takes a target-row window, hw_geom2d.trow0/ntrows).
    Pageable inputs are staged chunk by chunk through pinned buffers.
    `_marks` (tools/e2e_timeline.py): a list that receives (label, timing
    event) pairs for every upload, kernel and download; `_interleave` /
    `_pinned` override the launch order / input kind (tools/e2e_order.py)."""
    import torch

    timing = _marks is not None

    dev = torch.device("cuda", torch.cuda.current_device())
    nsrc = uh.shape[0]
    tp = flip(parity)
    shp_u, shp_v = _target_shape2d(grid, parity, m, m), _target_shape2d(grid, parity, m - 1, m - 1)
    ntx = shp_u[0]
    with warnings.catch_warnings():  # (read-only Field values: the tensors are only copy sources)
        warnings.simplefilter("ignore", UserWarning)
        srcs = [torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)) for a in (uh, vh)]
    u = torch.empty(uh.shape, dtype=torch.float64, device=dev)
    v = torch.empty(vh.shape, dtype=torch.float64, device=dev)
    ud = torch.empty(shp_u, dtype=torch.float64, device=dev)
    vd = torch.empty(shp_v, dtype=torch.float64, device=dev)
    ho_u = torch.empty(shp_u, dtype=torch.float64, pin_memory=True)
    ho_v = torch.empty(shp_v, dtype=torch.float64, pin_memory=True)
    comp = torch.cuda.current_stream(dev)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    s_in.wait_stream(comp)
    off = 0 if parity == PRIMAL else -1
    # chunk boundaries: nchunks equal chunks, or explicit fractions of the rows
    fr = np.linspace(0.0, 1.0, nchunks + 1) if np.isscalar(nchunks) else np.asarray(nchunks, dtype=float)
    edges = np.unique(np.round(fr * nsrc).astype(int))
    ranges = list(zip(edges[:-1], edges[1:]))
    if off == 0:
        # from primal data a target chunk also reads the first row of the next
        # chunk: upload it with this one (one duplicated row per chunk, same
        # bytes to the same place) so chunk k waits on upload k alone
        ranges = [(a, min(b + 1, nsrc)) for a, b in ranges]
    if grid.periodic and off < 0:
        # the first target rows read the last source row (periodic wrap):
        # send that row ahead of the chunks so the first launch need not wait
        # for the whole upload
        ranges.insert(0, (nsrc - 1, nsrc))
    # pageable sources (what a hermwave caller passes) go through pinned
    # staging buffers chunk by chunk: the host copy of chunk k + 1 (torch's
    # multithreaded CPU copy) overlaps the DMA of chunk k, where a pageable
    # copy_ would block the host thread for the whole synchronous upload
    pinned = all(x.is_pinned() for x in srcs) if _pinned is None else _pinned
    stage = srcs if pinned else [torch.empty(x.shape, dtype=torch.float64, pin_memory=True) for x in srcs]

    dt = cfg.dt(min(grid.hx, grid.hy))
    cap = -1 if cfg.stage_cap is None else int(cfg.stage_cap)
    tedges = np.unique(np.round(fr * ntx).astype(int))

    def plan():
        # first[r]: index of the earliest upload that carries source row r
        first = np.full(nsrc, -1, dtype=np.int64)
        for i, (a, b) in enumerate(ranges):
            seg = first[a:b]
            seg[seg < 0] = i
        # target chunks and the last upload each one needs (uploads complete in
        # issue order on one stream: waiting on that one covers the rest); this
        # host work runs once the first upload is on its way
        tchunks = []
        for t0, t1 in zip(tedges[:-1], tedges[1:]):
            if t1 <= t0:
                continue
            ends = [min(max(r % nsrc if grid.periodic else r, 0), nsrc - 1) for r in (t0 + off, t1 + off)]
            lo, hi = max(t0 + off, 0), min(t1 + off, nsrc - 1)
            k = max(int(first[ends].max()), int(first[lo:hi + 1].max()) if hi >= lo else -1)
            tchunks.append((int(t0), int(t1), k))
        return tchunks

    def launch(t0, t1, ev):
        comp.wait_event(ev)
        g = geom2d(grid, parity, bc, t0, t1 - t0)
        L.check(L.lib().hw_diss2d_half_step(C.byref(rows2d(u)), C.byref(rows2d(v)), ptr(ud) + 8 * t0 * shp_u[1] *
                                            (m + 1) ** 2, ptr(vd) + 8 * t0 * shp_v[1] * m * m, int(m), C.byref(g),
                                            dt, grid.hx, grid.hy, cfg.speed, cap, comp.cuda_stream), "half_step_2d")
        done = torch.cuda.Event(enable_timing=timing)
        done.record(comp)
        s_out.wait_event(done)
        with torch.cuda.stream(s_out):
            ho_u[t0:t1].copy_(ud[t0:t1], non_blocking=True)
            ho_v[t0:t1].copy_(vd[t0:t1], non_blocking=True)
        if timing:
            back = torch.cuda.Event(enable_timing=True)
            back.record(s_out)
            _marks.extend([(f"kern {t0}:{t1}", done), (f"down {t0}:{t1}", back)])

    # launch order (tools/e2e_order.py, C2 1024^2 m = 4): pinned sources issue
    # every upload first (5.1 GDOF/s; interleaved launches 4.7-5.2), staged
    # pageable sources launch each target chunk as soon as its uploads are
    # issued (3.3-3.4 GDOF/s against 2.6-2.7 uploads-first; the one-shot
    # driver-staged pageable copy of round 1 gave 1.1)
    interleave = (not pinned) if _interleave is None else bool(_interleave)
    arrived, nxt, tchunks = [], 0, None
    for i, (a, b) in enumerate(ranges):
        if not pinned:
            for x, hs in zip(srcs, stage):
                hs[a:b].copy_(x[a:b])
        with torch.cuda.stream(s_in):
            u[a:b].copy_(stage[0][a:b], non_blocking=True)
            v[a:b].copy_(stage[1][a:b], non_blocking=True)
            ev = torch.cuda.Event(enable_timing=timing)
            ev.record(s_in)
        arrived.append(ev)
        if timing:
            _marks.append((f"up {a}:{b}", ev))
        if tchunks is None:
            tchunks = plan()
        # launch every target chunk whose source rows are now on their way
        while interleave and nxt < len(tchunks) and tchunks[nxt][2] <= i:
            t0, t1, k = tchunks[nxt]
            launch(t0, t1, arrived[k])
            nxt += 1
    for t0, t1, k in tchunks[nxt:]:
        launch(t0, t1, arrived[k])
    s_out.synchronize()
    comp.wait_stream(s_out)
    return dt, ho_u.numpy(), ho_v.numpy()


def half_step_2d(state: FieldPair, cfg: SchemeConfig, bc: BoundarySpec2D) -> FieldPair:
    """Advance 2D (u, v) by dt/2 onto the opposite grid (dissipative.py:215-247)."""
    m = cfg.m
    grid = state.u.grid
    if state.u.orders != (m, m):
        raise ValueError(f"state carries orders {state.u.orders}, config wants ({m}, {m})")
    for spec in (bc.x, bc.y):
        check_periodicity(spec, grid.periodic)
    if isinstance(state.u.values, np.ndarray) and isinstance(state.v.values, np.ndarray) and \
            state.u.values.shape[0] >= 64:
        require_cuda()
        dt, hu, hv = _diss2d_host_pipelined(state.u.values, state.v.values, grid, state.parity, m, cfg, bc)
        t_new = state.time + 0.5 * dt
        parity = flip(state.parity)
        return FieldPair(Field2D(grid, parity, t_new, hu), Field2D(grid, parity, t_new, hv))
    st = Staging(state.u.values, state.v.values)
    u = st.to_dev(state.u.values)
    v = st.to_dev(state.v.values)
    ud = st.empty(_target_shape2d(grid, state.parity, m, m))
    vd = st.empty(_target_shape2d(grid, state.parity, m - 1, m - 1))
    dt = diss2d_into(u, v, ud, vd, grid, state.parity, m, cfg, bc, st.stream)
    t_new = state.time + 0.5 * dt
    parity = flip(state.parity)
    return FieldPair(Field2D(grid, parity, t_new, st.out(ud)), Field2D(grid, parity, t_new, st.out(vd)))


def advance_2d(state: FieldPair, cfg: SchemeConfig, bc: BoundarySpec2D, nhalf: int) -> FieldPair:
    """nhalf successive half_step_2d calls on device-resident buffers.

    Equivalent to ``for _ in range(nhalf): state = half_step_2d(state, cfg, bc)``
    (driver.py:400-401) including the float time accumulation, but with no
    host round trips: inputs are staged once and two buffer pairs alternate.
    """
    m = cfg.m
    grid = state.u.grid
    if state.u.orders != (m, m):
        raise ValueError(f"state carries orders {state.u.orders}, config wants ({m}, {m})")
    if nhalf <= 0:
        return state
    st = Staging(state.u.values, state.v.values)
    u = st.to_dev(state.u.values)
    v = st.to_dev(state.v.values)
    parity, t = state.parity, state.time
    owned = st.host  # staged copies of host inputs may be overwritten
    dst = {}
    for _ in range(nhalf):
        tp = flip(parity)
        if tp not in dst:
            dst[tp] = (st.empty(_target_shape2d(grid, parity, m, m)),
                       st.empty(_target_shape2d(grid, parity, m - 1, m - 1)))
        ud, vd = dst[tp]
        dt = diss2d_into(u, v, ud, vd, grid, parity, m, cfg, bc, st.stream)
        t = t + 0.5 * dt
        if owned:
            dst[parity] = (u, v)
        u, v, parity, owned = ud, vd, tp, True
    return FieldPair(Field2D(grid, parity, t, st.out(u)), Field2D(grid, parity, t, st.out(v)))


# ---------------------------------------------------------------- conservative

def cons2d_into(cur, prev, out, grid, parity_cur, m, cfg, bc, stream=None):
    dt = cfg.dt(min(grid.hx, grid.hy))
    g = geom2d(grid, parity_cur, bc)
    s = stream if stream is not None else stream_handle(cur.device)
    L.check(L.lib().hw_cons2d_step(C.byref(rows2d(cur)), ptr(prev), ptr(out), int(m), C.byref(g), dt,
                                   grid.hx, grid.hy, cfg.speed, s), "full_step_conservative")
    return dt


def cons1d_into(cur, prev, out, grid, parity_cur, m, cfg, bc: BoundarySpec, stream=None):
    check_periodicity(bc, grid.periodic)
    s = stream if stream is not None else stream_handle(cur.device)
    abc = L.axis_bc(bc)
    L.check(L.lib().hw_cons1d_step(ptr(cur), ptr(prev), ptr(out), int(m), grid.n_nodes(parity_cur),
                                   _PARITY[parity_cur], C.byref(abc), float(cfg.lam), s),
            "full_step_conservative")


def full_step_conservative(state: TwoLevelState, cfg: SchemeConfig, bc) -> TwoLevelState:
    """One conservative update (conservative.py:139-157): the new level lands
    on the previous level's grid; the old current becomes the new previous."""
    cur = state.current
    t_new = cur.time + 0.5 * cfg.dt(_min_h(cur))
    st = Staging(cur.values, state.previous.values)
    c = st.to_dev(cur.values)
    p = st.to_dev(state.previous.values)
    out = st.empty(tuple(state.previous.values.shape))
    if isinstance(cur, Field1D):
        m = cur.order
        if m != cfg.m:
            raise ValueError(f"state carries order {m}, config wants {cfg.m}")
        cons1d_into(c, p, out, cur.grid, cur.parity, m, cfg, bc, st.stream)
    else:
        m = cur.orders[0]
        if cur.orders != (cfg.m, cfg.m):
            raise ValueError(f"state carries orders {cur.orders}, config wants ({cfg.m}, {cfg.m})")
        cons2d_into(c, p, out, cur.grid, cur.parity, m, cfg, bc, st.stream)
    new = state.previous.with_values(st.out(out), time=t_new)
    return TwoLevelState(current=new, previous=cur)


def advance_conservative(state: TwoLevelState, cfg: SchemeConfig, bc, nsteps: int) -> TwoLevelState:
    """nsteps full_step_conservative calls in place on two device buffers
    (the update is element-wise in `previous`, conservative.py:127,136)."""
    if nsteps <= 0:
        return state
    cur, prev = state.current, state.previous
    st = Staging(cur.values, prev.values)
    a = st.to_dev(cur.values).clone() if not st.host else st.to_dev(cur.values)
    b = st.to_dev(prev.values).clone() if not st.host else st.to_dev(prev.values)
    pa, pb = cur.parity, prev.parity
    ta, tb = cur.time, prev.time
    grid = cur.grid
    for _ in range(nsteps):
        t_new = ta + 0.5 * cfg.dt(_min_h(cur))
        if isinstance(cur, Field1D):
            cons1d_into(a, b, b, grid, pa, cfg.m, cfg, bc, st.stream)
        else:
            cons2d_into(a, b, b, grid, pa, cfg.m, cfg, bc, st.stream)
        a, b = b, a
        pa, pb = pb, pa
        ta, tb = t_new, ta
    F = type(cur)
    return TwoLevelState(current=F(grid, pa, ta, st.out(a)), previous=F(grid, pb, tb, st.out(b)))


def bootstrap_first_half(g0, g1, cfg: SchemeConfig, bc) -> TwoLevelState:
    """Two starting levels from t=0 data (conservative.py:166-195)."""
    st = Staging(g0.values, g1.values)
    a = st.to_dev(g0.values)
    b = st.to_dev(g1.values)
    if isinstance(g0, Field1D):
        grid = g0.grid
        h = grid.h
        dt = cfg.dt(h)
        check_periodicity(bc, grid.periodic)
        nt = grid.n_nodes(flip(g0.parity))
        out = st.empty((nt, cfg.m + 1))
        abc = L.axis_bc(bc)
        L.check(L.lib().hw_boot1d(ptr(a), ptr(b), ptr(out), int(cfg.m), grid.n_nodes(g0.parity),
                                  _PARITY[g0.parity], C.byref(abc), dt, h, cfg.speed, st.stream),
                "bootstrap_first_half")
    else:
        grid = g0.grid
        dt = cfg.dt(min(grid.hx, grid.hy))
        g = geom2d(grid, g0.parity, bc)
        out = st.empty(_target_shape2d(grid, g0.parity, cfg.m, cfg.m))
        L.check(L.lib().hw_boot2d(C.byref(rows2d(a)), C.byref(rows2d(b)), ptr(out), int(cfg.m), C.byref(g),
                                  dt, grid.hx, grid.hy, cfg.speed, st.stream), "bootstrap_first_half")
    current = g0.with_values(st.out(out), parity=flip(g0.parity), time=g0.time + 0.5 * dt)
    return TwoLevelState(current=current, previous=g0)


# ---------------------------------------------------------------- 1D dissipative

def _forcing_table(forcing, cfg, grid, parity_src, dt, smax, t0):
    """Host evaluation of the user forcing callable (dissipative.py:102-105):
    F[s-1][l][t] = h^l dt^s/(l! s!) f(l, s-1, x_t, t0) for every coefficient
    l < 2m of the velocity interpolant (the reference loops over its full
    length, dissipative.py:102)."""
    m = cfg.m
    lv = 2 * m
    centers = grid.nodes(flip(parity_src))
    h = grid.h
    tab = np.zeros((smax, lv, len(centers)))
    fact = lambda n: float(np.prod(np.arange(2, n + 1))) if n > 1 else 1.0  # noqa: E731
    for s in range(1, smax + 1):
        for l in range(lv):
            fac = h**l * dt**s / (fact(l) * fact(s))
            tab[s - 1, l] = fac * np.broadcast_to(forcing(l, s - 1, centers, t0), centers.shape)
    return tab


def half_step_1d(state: FieldPair, cfg: SchemeConfig, bc: BoundarySpec, forcing=None) -> FieldPair:
    """Advance 1D (u, v) by dt/2 onto the opposite grid (dissipative.py:160-181)."""
    m = cfg.m
    grid = state.u.grid
    if state.u.order != m:
        raise ValueError(f"state carries order {state.u.order}, config wants {m}")
    check_periodicity(bc, grid.periodic)
    dt = cfg.dt(grid.h)
    st = Staging(state.u.values, state.v.values)
    u = st.to_dev(state.u.values)
    v = st.to_dev(state.v.values)
    nt = grid.n_nodes(flip(state.parity))
    ud = st.empty((nt, m + 1))
    vd = st.empty((nt, m))
    smax = cfg.stages_1d()
    f_dev = None
    if forcing is not None:
        f_dev = st.to_dev(_forcing_table(forcing, cfg, grid, state.parity, dt, smax, state.time)) \
            if st.host else None
        if f_dev is None:
            import torch

            f_dev = torch.as_tensor(_forcing_table(forcing, cfg, grid, state.parity, dt, smax, state.time),
                                    device=st.device)
    abc = L.axis_bc(bc)
    L.check(L.lib().hw_diss1d_half_step(ptr(u), ptr(v), ptr(ud), ptr(vd), int(m), grid.n_nodes(state.parity),
                                        _PARITY[state.parity], C.byref(abc), dt, grid.h, cfg.speed, int(smax),
                                        ptr(f_dev) if f_dev is not None else None, st.stream),
            "half_step_1d")
    t_new = state.time + 0.5 * dt
    parity = flip(state.parity)
    return FieldPair(Field1D(grid, parity, t_new, st.out(ud)), Field1D(grid, parity, t_new, st.out(vd)))


def interp_matrix(mu: int) -> np.ndarray:
    """interp.py:51-75, computed exactly by the library (read-only array)."""
    if not 0 <= mu <= 12:
        raise ValueError(f"interpolation order must be in [0, 12], got {mu}")
    out = np.empty((2 * mu + 2, 2 * mu + 2))
    L.check(L.lib().hw_interp_matrix(int(mu), out.ctypes.data_as(C.c_void_p)), "interp_matrix")
    out.setflags(write=False)
    return out


def require_finite(*arrays) -> None:
    """driver.py:259-262 _require_finite with the count done on the device."""
    from .device import Staging as _S

    for a in arrays:
        st = _S(a)
        d = st.to_dev(a)
        cnt = C.c_int64(0)
        L.check(L.lib().hw_count_nonfinite(ptr(d), int(d.numel()), C.byref(cnt), st.stream), "finite check")
        if cnt.value:
            raise NumericalError("non-finite field data detected")


class NumericalError(RuntimeError):
    """NaN or overflow detected in field data during a run (driver.py:46-47)."""


require_cuda  # re-exported for callers that want an early, explicit device check
