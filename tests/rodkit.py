"""Test helpers: hand-built single/multi-rod workloads (input layout only)."""
import dataclasses

import numpy as np

import workloads as W


def rod(N=10, L=1.0, r=0.01, E=1e6, rho=1000.0, Q=None, base=(0, 0, 0), clamp=-1, tip=None,
        nu=0.0, g=(0, 0, 0), dt=1e-5, n_steps=1, alpha_c=4.0 / 3.0, G=None, **extra):
    Q = np.eye(3) if Q is None else np.asarray(Q, float)
    n = np.array([N], np.int32)
    lhat = np.full(1, L / N)
    mat = W._rod_material(1, r, E, rho=rho, alpha_c=alpha_c)
    if G is not None:
        mat["shear_mod"] = np.array([G], float)
    pos = W.straight_rods(n, lhat, np.array([base], float), Q[2][None, :])
    w = W.Workload("rod", n, np.full(N, L / N), **mat, positions=pos, velocities=np.zeros_like(pos),
                   directors=np.tile(Q, (N, 1, 1)), omega=np.zeros((N, 3)),
                   clamp=np.array([clamp], np.int8), gravity=np.array(g, float),
                   damping=np.array([nu], float),
                   tip_force=None if tip is None else np.array([tip], float), dt=dt, n_steps=n_steps)
    return dataclasses.replace(w, **extra) if extra else w


def concat(ws):
    """Concatenate single-rod workloads into one batch (layout only)."""
    def cat(name, axis0=True):
        vals = [getattr(w, name) for w in ws]
        if all(v is None for v in vals):
            return None
        return np.concatenate(vals, axis=0)
    base = ws[0]
    out = dataclasses.replace(
        base, name="batch", n_elems=cat("n_elems"), rest_lengths=cat("rest_lengths"),
        density=cat("density"), area=cat("area"), I1=cat("I1"), I2=cat("I2"), youngs=cat("youngs"),
        shear_mod=cat("shear_mod"), alpha_c=cat("alpha_c"), positions=cat("positions"),
        velocities=cat("velocities"), directors=cat("directors"), omega=cat("omega"),
        clamp=cat("clamp"), damping=cat("damping"), tip_force=cat("tip_force"),
        rest_sigma=cat("rest_sigma"), rest_kappa=cat("rest_kappa"), act_A=cat("act_A"),
        act_f=cat("act_f"), act_L=cat("act_L"), magnetization=cat("magnetization"))
    return out
