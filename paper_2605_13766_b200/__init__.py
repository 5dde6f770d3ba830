"""paper_2605_13766_b200 -- B200-native batched discrete Cosserat rod stepping (arxiv 2605.13766).

Thin ctypes binding of the C-ABI in include/er.h (libelasticarod.so, built in-tree by
`build.py`).  Argument marshalling only: every step of the rod update runs in the CUDA
kernels of csrc/.  There is no CPU fallback: importing this package on a machine without
the built library, or calling it without a CUDA device, raises.

Names follow the C-ABI (north_star): er_create_batch, er_set_bc, er_set_forcing, er_step,
er_get_state, plus er_diagnostics / er_fault / er_set_option / er_query / er_destroy.
`RodBatch` wraps them for numpy / torch arrays.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ER_LIB") or os.path.join(_HERE, "lib", "libelasticarod.so")  # ER_LIB: A/B builds

ER_OK, ER_EINVAL, ER_EUNSTABLE, ER_EIO, ER_ENOMEM, ER_ECUDA = range(6)
ER_HOST, ER_DEVICE = 0, 1
ER_F_NONFINITE, ER_F_DEGENERATE, ER_F_ANTIPODAL, ER_F_OVERSPEED, ER_F_CONTACT = 1, 2, 4, 8, 16
ER_OPT_STEPS_PER_LAUNCH, ER_OPT_KERNEL, ER_OPT_PHASE_TIMING, ER_OPT_SWEEPS_PER_LAUNCH = 1, 2, 3, 4
ER_DEFAULT_SWEEPS = 0  # include/er.h: automatic (128 for small batches, else 1)
ER_NDIAG = 12
DIAG_NAMES = ("ke_trans", "ke_rot", "pe_shear", "pe_bend", "pe_grav", "pe_tip",
              "px", "py", "pz", "vmax", "mass", "n_elems")
ER_MAX_ELEMS_PER_ROD = 4095
ER_TILE_MAX_ELEMS = 511
_STATUS = {0: "ER_OK", 1: "ER_EINVAL", 2: "ER_EUNSTABLE", 3: "ER_EIO", 4: "ER_ENOMEM", 5: "ER_ECUDA"}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_bp = C.POINTER(C.c_int8)


class er_batch_desc(C.Structure):
    _fields_ = [
        ("n_rods", C.c_int32), ("n_elems", _ip), ("material_per_rod", C.c_int32),
        ("density", _dp), ("area", _dp), ("I1", _dp), ("I2", _dp), ("youngs", _dp),
        ("shear_mod", _dp), ("alpha_c", _dp), ("rest_lengths", _dp), ("rest_sigma", _dp),
        ("rest_kappa", _dp), ("positions", _dp), ("velocities", _dp), ("directors", _dp),
        ("omega", _dp), ("t0", C.c_double), ("src_mem", C.c_int32), ("device", C.c_int32),
        ("stream", C.c_void_p), ("tile_slots", C.c_int32),
    ]


class er_forcing(C.Structure):
    _fields_ = [
        ("gravity", C.c_double * 3), ("damping", _dp), ("damping_all", C.c_double),
        ("tip_force", _dp), ("act_A", _dp), ("act_f", _dp), ("act_L", _dp),
        ("act_component", C.c_int32), ("magnetization", _dp), ("b_field", C.c_double * 3),
        ("b_omega", C.c_double), ("b_axis", C.c_double * 3),
        ("musc_A", _dp), ("musc_T", _dp), ("musc_lambda", _dp), ("musc_phi", _dp), ("musc_component", C.c_int32),
    ]


class er_info(C.Structure):
    _fields_ = [
        ("n_rods", C.c_int64), ("n_elems_total", C.c_int64), ("n_nodes_total", C.c_int64),
        ("n_voronoi_total", C.c_int64), ("n_tiles", C.c_int64), ("tile_slots", C.c_int32),
        ("device", C.c_int32), ("stream", C.c_void_p), ("launches", C.c_int64),
        ("device_bytes", C.c_int64), ("t", C.c_double), ("bytes_per_step", C.c_double),
        ("warp_rod_elems", C.c_int32), ("warp_buffers", C.c_int32),
        ("shared_material", C.c_int32), ("reserved_", C.c_int32),
    ]


class er_contact(C.Structure):
    _fields_ = [
        ("enable", C.c_int32), ("k_n", C.c_double), ("gamma_n", C.c_double), ("mu_s", C.c_double),
        ("mu_k", C.c_double), ("v_stick", C.c_double), ("radius", _dp), ("exclude", C.c_int32),
        ("plane_on", C.c_int32), ("plane_n", C.c_double * 3), ("plane_d", C.c_double),
        ("cell0", C.c_double), ("n_levels", C.c_int32), ("pool_factor", C.c_double),
        ("skin", C.c_double),
    ]


class er_contact_stats(C.Structure):
    _fields_ = [
        ("candidates", C.c_int64), ("contacts", C.c_int64), ("cross_level", C.c_int64),
        ("plane_contacts", C.c_int64), ("pool_used", C.c_int64), ("list_entries", C.c_int64),
        ("scanned", C.c_int64), ("long_lists", C.c_int64), ("builds", C.c_int64),
        ("n_levels", C.c_int32), ("level_mask", C.c_int32), ("cell0", C.c_double), ("skin", C.c_double),
    ]


class er_phase_times(C.Structure):
    _fields_ = [("step_kernel_ms", C.c_double), ("step_kernel_launches", C.c_int64),
                ("contact_ms", C.c_double), ("contact_evals", C.c_int64)]


EXPORTS = ("er_create_batch", "er_set_bc", "er_set_forcing", "er_step", "er_get_state", "er_set_state",
           "er_diagnostics", "er_fault", "er_set_option", "er_set_trace", "er_query", "er_last_error",
           "er_abi_version", "er_destroy", "er_set_contact", "er_get_contact_stats", "er_get_phase_times",
           "er_set_external_loads", "er_set_contact_ghosts", "er_step_begin", "er_step_finish",
           "er_contact_records", "er_set_ghost_records")


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_2605_13766_b200/build.py` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    h = C.c_void_p
    lib.er_create_batch.argtypes = [C.POINTER(er_batch_desc), C.POINTER(h)]
    lib.er_set_bc.argtypes = [h, _bp]
    lib.er_set_forcing.argtypes = [h, C.POINTER(er_forcing)]
    lib.er_step.argtypes = [h, C.c_int64, C.c_double]
    lib.er_get_state.argtypes = [h, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, _dp]
    lib.er_set_state.argtypes = [h, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, _dp]
    lib.er_diagnostics.argtypes = [h, _dp]
    lib.er_fault.argtypes = [h, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
    lib.er_set_option.argtypes = [h, C.c_int32, C.c_int64]
    lib.er_set_trace.argtypes = [h, C.c_void_p]
    lib.er_query.argtypes = [h, C.POINTER(er_info)]
    lib.er_last_error.argtypes = [h]
    lib.er_last_error.restype = C.c_char_p
    lib.er_set_contact.argtypes = [h, C.POINTER(er_contact)]
    lib.er_get_contact_stats.argtypes = [h, C.POINTER(er_contact_stats)]
    lib.er_get_phase_times.argtypes = [h, C.POINTER(er_phase_times)]
    lib.er_set_external_loads.argtypes = [h, C.c_int32, C.c_void_p, C.c_void_p]
    lib.er_set_contact_ghosts.argtypes = [h, C.c_int64, _ip, _dp, _dp, _dp, _dp]
    lib.er_step_begin.argtypes = [h, C.c_double]
    lib.er_step_finish.argtypes = [h, C.c_double]
    lib.er_contact_records.argtypes = [h, C.c_int32, C.c_void_p]
    lib.er_set_ghost_records.argtypes = [h, C.c_int32, C.c_void_p]
    lib.er_abi_version.restype = C.c_int32
    lib.er_destroy.argtypes = [h]
    lib.er_destroy.restype = None
    for name in ("er_create_batch", "er_set_bc", "er_set_forcing", "er_step", "er_get_state",
                 "er_set_state", "er_diagnostics", "er_fault", "er_set_option", "er_set_trace", "er_query",
                 "er_set_contact", "er_get_contact_stats", "er_get_phase_times", "er_set_external_loads",
                 "er_set_contact_ghosts", "er_step_begin", "er_step_finish", "er_contact_records",
                 "er_set_ghost_records"):
        getattr(lib, name).restype = C.c_int
    return lib


lib = _load()


class ErError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


# ------------------------------------------------------------------------- raw C-ABI calls
def er_create_batch(desc: er_batch_desc) -> C.c_void_p:
    out = C.c_void_p()
    st = lib.er_create_batch(C.byref(desc), C.byref(out))
    if st != ER_OK:
        raise ErError(st, lib.er_last_error(None).decode())
    return out


def _check(handle, st):
    if st != ER_OK:
        raise ErError(st, lib.er_last_error(handle).decode())


def er_set_bc(handle, clamp_end):
    _check(handle, lib.er_set_bc(handle, clamp_end))


def er_set_forcing(handle, forcing: er_forcing):
    _check(handle, lib.er_set_forcing(handle, C.byref(forcing)))


def er_step(handle, n_steps: int, dt: float):
    _check(handle, lib.er_step(handle, int(n_steps), float(dt)))


def er_get_state(handle, dst_mem, positions, velocities, directors, omega):
    t = C.c_double()
    _check(handle, lib.er_get_state(handle, dst_mem, positions, velocities, directors, omega, C.byref(t)))
    return t.value


def er_set_state(handle, src_mem, positions, velocities, directors, omega, t=None):
    tt = None if t is None else C.byref(C.c_double(float(t)))
    _check(handle, lib.er_set_state(handle, src_mem, positions, velocities, directors, omega, tt))


def er_diagnostics(handle) -> np.ndarray:
    out = np.zeros(ER_NDIAG)
    _check(handle, lib.er_diagnostics(handle, out.ctypes.data_as(_dp)))
    return out


def er_fault(handle):
    rod, bits = C.c_int64(), C.c_int32()
    _check(handle, lib.er_fault(handle, C.byref(rod), C.byref(bits)))
    return rod.value, bits.value


def er_set_option(handle, option: int, value: int):
    _check(handle, lib.er_set_option(handle, int(option), int(value)))


def er_set_trace(handle, device_ptr):
    _check(handle, lib.er_set_trace(handle, device_ptr))


def er_query(handle) -> er_info:
    info = er_info()
    _check(handle, lib.er_query(handle, C.byref(info)))
    return info


def er_set_contact(handle, contact):
    _check(handle, lib.er_set_contact(handle, None if contact is None else C.byref(contact)))


def er_set_contact_ghosts(handle, n, n_elems, radius, stiffness, lmin, lmax):
    _check(handle, lib.er_set_contact_ghosts(handle, n, n_elems, radius, stiffness, lmin, lmax))


def er_step_begin(handle, dt):
    _check(handle, lib.er_step_begin(handle, dt))


def er_step_finish(handle, dt):
    _check(handle, lib.er_step_finish(handle, dt))


def er_contact_records(handle, dst_mem, dst):
    _check(handle, lib.er_contact_records(handle, dst_mem, dst))


def er_set_ghost_records(handle, src_mem, src):
    _check(handle, lib.er_set_ghost_records(handle, src_mem, src))


def er_set_external_loads(handle, src_mem, node_force, elem_couple):
    _check(handle, lib.er_set_external_loads(handle, src_mem, node_force, elem_couple))


def er_get_contact_stats(handle) -> er_contact_stats:
    out = er_contact_stats()
    _check(handle, lib.er_get_contact_stats(handle, C.byref(out)))
    return out


def er_get_phase_times(handle) -> er_phase_times:
    out = er_phase_times()
    _check(handle, lib.er_get_phase_times(handle, C.byref(out)))
    return out


def er_destroy(handle):
    lib.er_destroy(handle)


# ------------------------------------------------------------------------- marshalling helpers
def _is_torch(a):
    return type(a).__module__.startswith("torch")


class _Keep:
    """Converts arrays to C pointers and keeps the converted buffers alive."""

    def __init__(self):
        self.refs = []

    def host(self, a, dtype=np.float64, ctype=_dp):
        if a is None:
            return None
        if _is_torch(a):
            a = a.detach().cpu().numpy()
        a = np.ascontiguousarray(a, dtype=dtype)
        self.refs.append(a)
        return a.ctypes.data_as(ctype)

    def any(self, a):
        """Host numpy/torch-cpu -> (ptr, ER_HOST); torch cuda tensor -> (device ptr, ER_DEVICE)."""
        if a is None:
            return None, None
        if _is_torch(a) and a.is_cuda:
            import torch
            if a.dtype != torch.float64 or not a.is_contiguous():
                a = a.to(torch.float64).contiguous()
            self.refs.append(a)
            return C.cast(C.c_void_p(a.data_ptr()), _dp), ER_DEVICE
        return self.host(a), ER_HOST


class RodBatch:
    """A batch of independent rods resident on one GPU.

    `w` is any object with the workload attributes of include/er.h (e.g. workloads.Workload):
    n_elems, rest_lengths, density, area, I1, I2, youngs, shear_mod, alpha_c, positions,
    velocities, directors, omega, and optional rest_sigma, rest_kappa, t0, clamp, gravity,
    damping, tip_force, act_A/act_f/act_L/act_component, magnetization/b_field/b_omega.
    State arrays may be numpy (host) or torch CUDA tensors (device)."""

    def __init__(self, w, device: int = 0, stream=None, apply_bc_forcing: bool = True, tile_slots: int = 0):
        k = _Keep()
        d = er_batch_desc()
        d.n_rods = int(len(w.n_elems))
        d.n_elems = k.host(w.n_elems, np.int32, _ip)
        d.material_per_rod = 1 if len(w.density) == d.n_rods else 0
        for name in ("density", "area", "I1", "I2", "youngs", "shear_mod", "alpha_c", "rest_lengths"):
            setattr(d, name, k.host(getattr(w, name)))
        d.rest_sigma = k.host(getattr(w, "rest_sigma", None))
        d.rest_kappa = k.host(getattr(w, "rest_kappa", None))
        mems = set()
        for name in ("positions", "velocities", "directors", "omega"):
            ptr, mem = k.any(getattr(w, name, None))
            setattr(d, name, ptr)
            if mem is not None:
                mems.add(mem)
        if len(mems) > 1:
            raise ValueError("state arrays must all be host or all be device")
        d.src_mem = mems.pop() if mems else ER_HOST
        d.t0 = float(getattr(w, "t0", 0.0))
        d.device = int(device)
        d.stream = None if stream is None else C.c_void_p(int(getattr(stream, "cuda_stream", stream)))
        d.tile_slots = int(tile_slots)
        if d.src_mem == ER_DEVICE:  # the library reads the arrays on its own stream: finish their producers
            import torch
            torch.cuda.current_stream(int(device)).synchronize()
        self.device = int(device)
        self.handle = er_create_batch(d)
        self.n_rods = d.n_rods
        info = er_query(self.handle)
        self.n_elems_total = info.n_elems_total
        self.n_nodes_total = info.n_nodes_total
        if apply_bc_forcing:
            self.set_bc(getattr(w, "clamp", None))
            self.set_forcing_from(w)
            if getattr(w, "contact", None) is not None:
                self.set_contact(w.contact)
            if getattr(w, "ext_force", None) is not None or getattr(w, "ext_couple", None) is not None:
                self.set_external_loads(getattr(w, "ext_force", None), getattr(w, "ext_couple", None))

    # -- boundary conditions / forcing
    def set_bc(self, clamp_end=None):
        k = _Keep()
        er_set_bc(self.handle, k.host(clamp_end, np.int8, _bp))

    def set_forcing(self, gravity=(0, 0, 0), damping=None, damping_all=0.0, tip_force=None,
                    act_A=None, act_f=None, act_L=None, act_component=0, magnetization=None,
                    b_field=(0, 0, 0), b_omega=0.0, b_axis=(0, 0, 0), musc_A=None, musc_T=None,
                    musc_lambda=None, musc_phi=None, musc_component=0):
        k = _Keep()
        f = er_forcing()
        f.gravity = (C.c_double * 3)(*[float(x) for x in gravity])
        f.damping = k.host(damping)
        f.damping_all = float(damping_all)
        f.tip_force = k.host(tip_force)
        f.act_A, f.act_f, f.act_L = k.host(act_A), k.host(act_f), k.host(act_L)
        f.act_component = int(act_component)
        f.magnetization = k.host(magnetization)
        f.b_field = (C.c_double * 3)(*[float(x) for x in (b_field if b_field is not None else (0, 0, 0))])
        f.b_omega = float(b_omega)
        f.b_axis = (C.c_double * 3)(*[float(x) for x in (b_axis if b_axis is not None else (0, 0, 0))])
        f.musc_A, f.musc_T = k.host(musc_A), k.host(musc_T)
        f.musc_lambda, f.musc_phi = k.host(musc_lambda), k.host(musc_phi)
        f.musc_component = int(musc_component)
        er_set_forcing(self.handle, f)

    def set_external_loads(self, node_force=None, elem_couple=None):
        """er_set_external_loads: node_force [n_nodes, 3] lab (N), elem_couple [n_elems, 3] local
        (N m), canonical order; numpy (host) or torch CUDA tensors (device), both the same kind;
        None clears that array."""
        k = _Keep()
        pf, mf = k.any(node_force)
        pc, mc = k.any(elem_couple)
        mems = {m for m in (mf, mc) if m is not None}
        if len(mems) > 1:
            raise ValueError("node_force and elem_couple must both be host or both be device")
        for a, rows in ((node_force, self.n_nodes_total), (elem_couple, self.n_elems_total)):
            if a is not None and tuple(a.shape) != (rows, 3):
                raise ValueError(f"external load of shape {tuple(a.shape)}, expected ({rows}, 3)")
        mem = mems.pop() if mems else ER_HOST
        if mem == ER_DEVICE:
            self._after_torch()
        er_set_external_loads(self.handle, mem, pf, pc)

    def set_forcing_from(self, w):
        self.set_forcing(gravity=getattr(w, "gravity", (0, 0, 0)), damping=getattr(w, "damping", None),
                         tip_force=getattr(w, "tip_force", None), act_A=getattr(w, "act_A", None),
                         act_f=getattr(w, "act_f", None), act_L=getattr(w, "act_L", None),
                         act_component=getattr(w, "act_component", 0),
                         magnetization=getattr(w, "magnetization", None),
                         b_field=getattr(w, "b_field", None), b_omega=getattr(w, "b_omega", 0.0),
                         b_axis=getattr(w, "b_axis", None), musc_A=getattr(w, "musc_A", None),
                         musc_T=getattr(w, "musc_T", None), musc_lambda=getattr(w, "musc_lambda", None),
                         musc_phi=getattr(w, "musc_phi", None), musc_component=getattr(w, "musc_component", 0))

    def set_contact(self, c=None, cell0: float = 0.0, n_levels: int = 0, pool_factor: float = 0.0,
                    skin: float = 0.0):
        """Enable rod-rod / half-space contact from an object with the attributes of
        workloads.Contact (k_n, gamma_n, mu_s, mu_k, v_stick, radius, exclude, plane_n, plane_d);
        None disables it."""
        if c is None:
            er_set_contact(self.handle, None)
            return
        k = _Keep()
        s = er_contact()
        s.enable = 1
        s.k_n, s.gamma_n = float(c.k_n), float(c.gamma_n)
        s.mu_s, s.mu_k, s.v_stick = float(c.mu_s), float(c.mu_k), float(c.v_stick)
        s.radius = k.host(getattr(c, "radius", None))
        s.exclude = int(c.exclude)
        pn = getattr(c, "plane_n", None)
        s.plane_on = 0 if pn is None else 1
        s.plane_n = (C.c_double * 3)(*([float(x) for x in pn] if pn is not None else [0.0, 0.0, 1.0]))
        s.plane_d = float(getattr(c, "plane_d", 0.0))
        s.cell0 = float(getattr(c, "cell0", cell0) or cell0)
        s.n_levels = int(getattr(c, "n_levels", n_levels) or n_levels)
        s.pool_factor = float(pool_factor)
        s.skin = float(skin)
        er_set_contact(self.handle, s)

    def set_contact_ghosts(self, n_elems, radius, stiffness, lhat_min, lhat_max):
        """Declare the ghost rods of a contact shard (include/er.h er_set_contact_ghosts); empty
        arrays remove them."""
        k = _Keep()
        n = int(len(n_elems))
        er_set_contact_ghosts(self.handle, n, k.host(n_elems, np.int32, _ip), k.host(radius), k.host(stiffness),
                              k.host(lhat_min), k.host(lhat_max))

    def step_begin(self, dt: float):
        er_step_begin(self.handle, dt)

    def step_finish(self, dt: float):
        er_step_finish(self.handle, dt)

    def contact_records(self, out):
        """Own node records after er_step_begin ([n_nodes][6]: r, v) into `out` (a torch CUDA
        tensor -> device copy, numpy -> host)."""
        dev = _is_torch(out) and out.is_cuda
        er_contact_records(self.handle, ER_DEVICE if dev else ER_HOST, out.data_ptr() if _is_torch(out) else out.ctypes.data)

    def set_ghost_records(self, src):
        dev = _is_torch(src) and src.is_cuda
        if dev:
            import torch
            torch.cuda.current_stream(self.device).synchronize()  # its producer ran on torch's stream
        buf = src if _is_torch(src) else np.ascontiguousarray(src, dtype=np.float64)
        er_set_ghost_records(self.handle, ER_DEVICE if dev else ER_HOST,
                             buf.data_ptr() if _is_torch(buf) else buf.ctypes.data)

    def contact_stats(self) -> er_contact_stats:
        return er_get_contact_stats(self.handle)

    def phase_times(self) -> er_phase_times:
        return er_get_phase_times(self.handle)

    # -- stepping / state
    def step(self, n_steps: int, dt: float):
        er_step(self.handle, n_steps, dt)

    def set_option(self, option: int, value: int):
        er_set_option(self.handle, option, value)

    def get_state(self):
        """Host copies (numpy) of positions, velocities, directors, omega and t."""
        pos = np.empty((self.n_nodes_total, 3))
        vel = np.empty((self.n_nodes_total, 3))
        dirs = np.empty((self.n_elems_total, 3, 3))
        om = np.empty((self.n_elems_total, 3))
        t = er_get_state(self.handle, ER_HOST, pos.ctypes.data, vel.ctypes.data, dirs.ctypes.data, om.ctypes.data)
        return pos, vel, dirs, om, t

    def get_state_into(self, positions=None, velocities=None, directors=None, omega=None):
        """Write the state into caller buffers (torch CUDA tensors -> device copy; numpy -> host)."""
        bufs = [positions, velocities, directors, omega]
        dev = any(b is not None and _is_torch(b) and b.is_cuda for b in bufs)
        ptrs = [None if b is None else (b.data_ptr() if _is_torch(b) else b.ctypes.data) for b in bufs]
        return er_get_state(self.handle, ER_DEVICE if dev else ER_HOST, *ptrs)

    def _after_torch(self):
        """Order the batch's stream after torch's current stream (device tensors handed to the
        library are read on the batch's stream)."""
        import torch
        cur = torch.cuda.current_stream(self.device)
        if cur.cuda_stream != (self.info().stream or 0):
            torch.cuda.ExternalStream(self.info().stream, device=self.device).wait_stream(cur)

    def set_state(self, positions=None, velocities=None, directors=None, omega=None, t=None):
        """Overwrite (parts of) the state; numpy -> host source, torch CUDA tensors -> device."""
        k = _Keep()
        bufs = [positions, velocities, directors, omega]
        dev = any(x is not None and _is_torch(x) and x.is_cuda for x in bufs)
        ptrs = [k.any(x)[0] if dev else k.host(x) for x in bufs]
        if dev:
            self._after_torch()
        er_set_state(self.handle, ER_DEVICE if dev else ER_HOST, *ptrs, t=t)

    def diagnostics(self) -> np.ndarray:
        return er_diagnostics(self.handle)

    def fault(self):
        return er_fault(self.handle)

    def info(self) -> er_info:
        return er_query(self.handle)

    def close(self):
        if getattr(self, "handle", None):
            er_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
