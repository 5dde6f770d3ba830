"""ctypes wrapper of the CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py
(`cpu_baseline` and `--impl reference`) may import this package.  The product
package `paper_2605_13766_b200` never imports it, and it never imports the
product package.  It consumes workloads.Workload arrays verbatim.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-Wall"]

NDIAG = 12
DIAG_NAMES = ("ke_trans", "ke_rot", "pe_shear", "pe_bend", "pe_grav", "pe_tip",
              "px", "py", "pz", "vmax", "mass", "n_elems")
F_NONFINITE, F_DEGENERATE, F_ANTIPODAL, F_OVERSPEED = 1, 2, 4, 8
SYNC, ASYNC = 0, 1


def build(force: bool = False, src: str = _SRC, out: str = _LIB) -> str:
    """Compile liboracle.so with gcc (plain C, no FMA contraction).

    The library is compiled to a per-process temporary file and renamed into place, so that
    concurrent builders (bench.py's cpu_baseline fan-out, pytest-xdist workers) never dlopen a
    half-written file: each sees either the old complete library or the new one."""
    hdr = os.path.join(os.path.dirname(src), "oracle.h")
    if force or not os.path.exists(out) or os.path.getmtime(out) < max(
            os.path.getmtime(src), os.path.getmtime(hdr)):
        tmp = f"{out}.tmp.{os.getpid()}"
        try:
            subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, src, "-lm"])
            os.replace(tmp, out)
        finally:
            if os.path.exists(tmp):
                os.unlink(tmp)
    return out


_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_bp = C.POINTER(C.c_int8)


class _Contact(C.Structure):
    _fields_ = [
        ("enable", C.c_int32), ("k_n", C.c_double), ("gamma_n", C.c_double), ("mu_s", C.c_double),
        ("mu_k", C.c_double), ("v_stick", C.c_double), ("radius", _dp), ("exclude", C.c_int32),
        ("plane_on", C.c_int32), ("plane_n", C.c_double * 3), ("plane_d", C.c_double),
    ]


class _Problem(C.Structure):
    _fields_ = [
        ("n_rods", C.c_int32), ("n_elems", _ip), ("material_per_rod", C.c_int32),
        ("density", _dp), ("area", _dp), ("I1", _dp), ("I2", _dp), ("youngs", _dp),
        ("shear_mod", _dp), ("alpha_c", _dp), ("rest_lengths", _dp), ("rest_sigma", _dp),
        ("rest_kappa", _dp), ("clamp", _bp), ("gravity", C.c_double * 3), ("damping", _dp),
        ("tip_force", _dp), ("act_A", _dp), ("act_f", _dp), ("act_L", _dp),
        ("act_component", C.c_int32), ("magnetization", _dp), ("b_field", C.c_double * 3),
        ("b_omega", C.c_double), ("b_axis", C.c_double * 3),
        ("musc_A", _dp), ("musc_T", _dp), ("musc_lambda", _dp), ("musc_phi", _dp), ("musc_component", C.c_int32),
        ("contact", C.POINTER(_Contact)), ("ext_force", _dp), ("ext_couple", _dp),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        # ER_ORACLE_LIB: a prebuilt oracle library (tools/oracle_mutants.py loads mutated builds)
        _lib = C.CDLL(os.environ.get("ER_ORACLE_LIB") or build())
        _lib.orc_rot.argtypes = [_dp, _dp]
        _lib.orc_logrot.argtypes = [_dp, _dp]
        _lib.orc_logrot.restype = C.c_int
        _lib.orc_ax.argtypes = [_dp, _dp]
        _lib.orc_skew.argtypes = [_dp, _dp]
        _lib.orc_rod_strains.argtypes = [C.c_int32, _dp, _dp, _dp, _dp, _dp, _dp]
        _lib.orc_rod_strains.restype = C.c_int
        _lib.orc_rod_loads.argtypes = [C.POINTER(_Problem), C.c_int32, _dp, _dp, _dp, _dp, C.c_double,
                                       _dp, _dp, _dp, _dp]
        _lib.orc_rod_loads.restype = C.c_int
        _lib.orc_step.argtypes = [C.POINTER(_Problem), _dp, _dp, _dp, _dp, _dp, C.c_int64, C.c_double,
                                  C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
        _lib.orc_step.restype = C.c_int
        _lib.orc_energy.argtypes = [C.POINTER(_Problem), _dp, _dp, _dp, _dp, C.c_double, _dp]
        _lib.orc_energy.restype = C.c_int
        _lib.orc_segment_closest.argtypes = [_dp, _dp, _dp, _dp, _dp, _dp, _dp]
        _lib.orc_contact_pairs.argtypes = [C.POINTER(_Problem), _dp, C.c_int64, C.POINTER(C.c_int64), _dp]
        _lib.orc_contact_pairs.restype = C.c_int64
        _lib.orc_contact_forces.argtypes = [C.POINTER(_Problem), _dp, _dp, _dp]
    return _lib


def _f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a


def _ptr(a, t=_dp):
    return None if a is None else a.ctypes.data_as(t)


class Problem:
    """Holds a ctypes orc_problem plus references keeping its arrays alive."""

    def __init__(self, w):
        self._keep = []
        per_rod = w.density.shape[0] == w.n_rods   # else per element [n_elems_total]

        def k(a, dtype=np.float64):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=dtype)
            self._keep.append(a)
            return a

        p = _Problem()
        p.n_rods = w.n_rods
        p.n_elems = _ptr(k(w.n_elems, np.int32), _ip)
        p.material_per_rod = 1 if per_rod else 0
        for name in ("density", "area", "I1", "I2", "youngs", "shear_mod", "alpha_c", "rest_lengths",
                     "rest_sigma", "rest_kappa", "damping", "tip_force", "act_A", "act_f", "act_L",
                     "magnetization", "musc_A", "musc_T", "musc_lambda", "musc_phi"):
            setattr(p, name, _ptr(k(getattr(w, name, None))))
        p.clamp = _ptr(k(w.clamp, np.int8), _bp)
        p.gravity = (C.c_double * 3)(*[float(x) for x in w.gravity])
        p.act_component = int(w.act_component)
        b = w.b_field if w.b_field is not None else np.zeros(3)
        p.b_field = (C.c_double * 3)(*[float(x) for x in b])
        p.b_omega = float(w.b_omega)
        ax = w.b_axis if getattr(w, "b_axis", None) is not None else np.zeros(3)
        p.b_axis = (C.c_double * 3)(*[float(x) for x in ax])
        p.musc_component = int(getattr(w, "musc_component", 0))
        ct = getattr(w, "contact", None)
        if ct is not None:
            c = _Contact()
            c.enable = 1
            c.k_n, c.gamma_n, c.mu_s, c.mu_k, c.v_stick = ct.k_n, ct.gamma_n, ct.mu_s, ct.mu_k, ct.v_stick
            c.radius = _ptr(k(ct.radius))
            c.exclude = int(ct.exclude)
            c.plane_on = 0 if ct.plane_n is None else 1
            c.plane_n = (C.c_double * 3)(*([float(x) for x in ct.plane_n] if ct.plane_n is not None else [0, 0, 1]))
            c.plane_d = float(ct.plane_d)
            self._keep.append(c)
            p.contact = C.pointer(c)
        p.ext_force = _ptr(k(getattr(w, "ext_force", None)))
        p.ext_couple = _ptr(k(getattr(w, "ext_couple", None)))
        self.c = p


# ------------------------------------------------------------------ SO(3) maps
def rot(v):
    v = _f64(v)
    R = np.empty(9)
    lib().orc_rot(_ptr(v), _ptr(R))
    return R.reshape(3, 3)


def logrot(R):
    R = _f64(R).reshape(9)
    v = np.empty(3)
    f = lib().orc_logrot(_ptr(R), _ptr(v))
    return v, f


def ax(U):
    U = _f64(U).reshape(9)
    v = np.empty(3)
    lib().orc_ax(_ptr(U), _ptr(v))
    return v


def skew(v):
    v = _f64(v)
    W = np.empty(9)
    lib().orc_skew(_ptr(v), _ptr(W))
    return W.reshape(3, 3)


def rod_strains(lhat, pos, dirs):
    lhat, pos, dirs = _f64(lhat), _f64(pos), _f64(dirs)
    N = lhat.shape[0]
    e, s, k = np.empty(N), np.empty((N, 3)), np.empty((max(N - 1, 0), 3))
    f = lib().orc_rod_strains(N, _ptr(lhat), _ptr(pos), _ptr(dirs), _ptr(e), _ptr(s), _ptr(k))
    return e, s, k, f


def rod_loads(w, rod, pos, vel, dirs, omega, t=0.0):
    """Per-rod loads; state arrays are the rod's own slices."""
    P = Problem(w)
    N = int(w.n_elems[rod])
    pos, vel, dirs, omega = _f64(pos), _f64(vel), _f64(dirs), _f64(omega)
    F, a = np.empty((N + 1, 3)), np.empty((N + 1, 3))
    Cc, al = np.empty((N, 3)), np.empty((N, 3))
    f = lib().orc_rod_loads(C.byref(P.c), rod, _ptr(pos), _ptr(vel), _ptr(dirs), _ptr(omega), t,
                            _ptr(F), _ptr(Cc), _ptr(a), _ptr(al))
    return dict(F=F, C=Cc, a=a, alpha=al, fault=f)


class State:
    def __init__(self, positions, velocities, directors, omega, t):
        self.positions = _f64(positions).copy()
        self.velocities = _f64(velocities).copy()
        self.directors = _f64(directors).copy()
        self.omega = _f64(omega).copy()
        self.t = float(t)

    @classmethod
    def of(cls, w):
        return cls(w.positions, w.velocities, w.directors, w.omega, w.t0)


def step(w, state: Optional[State] = None, n_steps: Optional[int] = None, dt: Optional[float] = None,
         protocol: int = SYNC):
    """Run n_steps of the oracle in place on `state` (a fresh copy of w's state if None).
    Returns (state, status, bad_rod, fault_bits)."""
    st = State.of(w) if state is None else state
    P = Problem(w)
    t = C.c_double(st.t)
    bad = C.c_int64(-1)
    bits = C.c_int32(0)
    status = lib().orc_step(C.byref(P.c), _ptr(st.positions), _ptr(st.velocities), _ptr(st.directors),
                            _ptr(st.omega), C.byref(t), int(w.n_steps if n_steps is None else n_steps),
                            float(w.dt if dt is None else dt), protocol, C.byref(bad), C.byref(bits))
    st.t = t.value
    return st, status, bad.value, bits.value


def energy(w, state: Optional[State] = None):
    st = State.of(w) if state is None else state
    P = Problem(w)
    out = np.empty(NDIAG)
    lib().orc_energy(C.byref(P.c), _ptr(st.positions), _ptr(st.velocities), _ptr(st.directors),
                     _ptr(st.omega), st.t, _ptr(out))
    return out


# ------------------------------------------------------------------ contact (NEXT-4)
def segment_closest(p0, p1, q0, q1):
    p0, p1, q0, q1 = (_f64(x) for x in (p0, p1, q0, q1))
    s, t, d = C.c_double(), C.c_double(), C.c_double()
    lib().orc_segment_closest(_ptr(p0), _ptr(p1), _ptr(q0), _ptr(q1), C.byref(s), C.byref(t), C.byref(d))
    return s.value, t.value, d.value


def contact_pairs(w, positions, max_pairs=1 << 20):
    """Exhaustive O(E^2) detection: element pairs (a < b) with gap < 0, and their gaps."""
    P = Problem(w)
    pos = _f64(positions)
    pairs = np.zeros((max_pairs, 2), np.int64)
    gaps = np.zeros(max_pairs)
    n = lib().orc_contact_pairs(C.byref(P.c), _ptr(pos), max_pairs, pairs.ctypes.data_as(C.POINTER(C.c_int64)),
                                _ptr(gaps))
    n = min(n, max_pairs)
    return pairs[:n], gaps[:n]


def contact_forces(w, positions, velocities):
    P = Problem(w)
    pos, vel = _f64(positions), _f64(velocities)
    F = np.zeros_like(pos)
    lib().orc_contact_forces(C.byref(P.c), _ptr(pos), _ptr(vel), _ptr(F))
    return F
