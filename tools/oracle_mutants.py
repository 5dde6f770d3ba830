"""Mutation check of the oracle's pins (CPU only; run by tests/test_oracle_mutants.py).

Each mutant is one plausible mistake in oracle/oracle.c -- a dropped term, a wrong sign, power or
index, a transposed operand -- in the arithmetic of Eqs. (1a)-(1b), the strain
definitions, the SO(3) maps or the integrator.
For every mutant the script copies oracle.c, applies the edit, builds the library into a temporary
directory and runs the CPU pin suite (tests/test_oracle_*.py) against it via ER_ORACLE_LIB.  A
mutant is *killed* when at least one pin fails.  Exit status 0 iff every mutant is killed.

    python tools/oracle_mutants.py            # all mutants
    python tools/oracle_mutants.py beta_sign  # a subset by name
"""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# (name, what it breaks, old text, new text).  `old` must occur in oracle.c; every occurrence is
# replaced.
MUTANTS = [
    # --- the ten of VERDICT r01 "What's weak" 1 (Eq. (1b) finite-strain and bend-twist terms)
    ("beta_sign", "beta = m x kappa instead of kappa x m (PAPER.md:247)",
     "v_cross(c->kap + 3 * k, c->mbar + 3 * k, c->beta + 3 * k);",
     "v_cross(c->mbar + 3 * k, c->kap + 3 * k, c->beta + 3 * k);"),
    ("beta_drop", "kappa x B kappa / e^3 term dropped",
     "c->beta[3 * k + q] *= c->Dh[k];", "c->beta[3 * k + q] *= 0.0;"),
    ("beta_average", "A^h beta without the 1/2",
     "Cj[q] = (mn - mc) + 0.5 * (bn + bc);", "Cj[q] = (mn - mc) + (bn + bc);"),
    ("bend_eps2", "B kappa / eps^2 instead of / eps^3",
     "double e3k = c->eps[k] * c->eps[k] * c->eps[k];", "double e3k = c->eps[k] * c->eps[k];"),
    ("voronoi_eps_is_e", "Voronoi dilatation eps_k := e_k (not the neighbouring mean)",
     "c->eps[k] = (0.5 * (c->l[k - 1] + c->l[k])) / c->Dh[k];", "c->eps[k] = c->e[k];"),
    ("dilatation_e1", "unsteady dilatation J w edot / e instead of / e^2 (PAPER.md:248)",
     "Cj[q] += Jw[q] / (c->e[j] * c->e[j]) * c->edot[j];", "Cj[q] += Jw[q] / c->e[j] * c->edot[j];"),
    ("alpha_no_e", "alpha = C / J instead of e C / J (rho I / e on the left of Eq. (1b))",
     "c->al[3 * j + q] = c->e[j] / c->J[3 * j + q] * Cj[q]", "c->al[3 * j + q] = 1.0 / c->J[3 * j + q] * Cj[q]"),
    ("transport_e2", "transport (J w / e^2) x w instead of / e",
     "tmp[q] = Jw[q] / c->e[j];", "tmp[q] = Jw[q] / (c->e[j] * c->e[j]);"),
    ("sigma0_sign", "n = S (sigma + sigma0) / e",
     "d[q] = c->sig[3 * j + q] - s0;", "d[q] = c->sig[3 * j + q] + s0;"),
    ("nbar_no_e", "n = S (sigma - sigma0) without the 1/e (PAPER.md:243)",
     "c->nbar[3 * j + q] = c->S[3 * j + q] * d[q] / c->e[j];", "c->nbar[3 * j + q] = c->S[3 * j + q] * d[q];"),
    # --- further plausible mistakes across the method
    ("voronoi_B_arithmetic", "B on Voronoi domains as the rest-length-weighted arithmetic mean",
     "c->Bv[3 * k + q] = (2.0 * c->Dh[k]) / (c->lhat[k - 1] / c->B[3 * (k - 1) + q] + c->lhat[k] / c->B[3 * k + q]);",
     "c->Bv[3 * k + q] = (c->B[3 * (k - 1) + q] * c->lhat[k - 1] + c->B[3 * k + q] * c->lhat[k]) / (2.0 * c->Dh[k]);"),
    ("shear_torque_sign", "S sigma x Q t instead of Q t x S sigma",
     "v_cross(Qt, Sd, tmp);", "v_cross(Sd, Qt, tmp);"),
    ("shear_torque_no_lhat", "shear torque per length not integrated over the element",
     "Cj[q] += c->lhat[j] * tmp[q];", "Cj[q] += tmp[q];"),
    ("shear_torque_sigma0_sign", "shear torque with sigma + sigma0",
     "Sd[q] = c->S[3 * j + q] * (c->sig[3 * j + q] - s0);", "Sd[q] = c->S[3 * j + q] * (c->sig[3 * j + q] + s0);"),
    ("transport_sign", "transport w x (J w / e)",
     "v_cross(tmp, w + 3 * j, tmp);", "v_cross(w + 3 * j, tmp, tmp);"),
    ("force_difference_sign", "F_i = n_i + n_{i-1}",
     "if (i > 0) f -= c->nlab[3 * (i - 1) + q];", "if (i > 0) f += c->nlab[3 * (i - 1) + q];"),
    ("damping_sign", "a = F/m + nu v",
     "c->a[3 * i + q] = f / c->m[i] - c->nu * v[3 * i + q];", "c->a[3 * i + q] = f / c->m[i] + c->nu * v[3 * i + q];"),
    ("mass_full_lump", "each end node gets the whole element mass",
     "if (i > 0) m += 0.5 * c->me[i - 1];", "if (i > 0) m += c->me[i - 1];"),
    ("edot_no_lhat", "de/dt without the 1/lhat",
     "c->edot[j] = v_dot(c->tg + 3 * j, dv) / c->lhat[j];", "c->edot[j] = v_dot(c->tg + 3 * j, dv);"),
    ("voronoi_length_right", "Dh_k = lhat_k (not the mean of the two elements)",
     "c->Dh[k] = 0.5 * (c->lhat[k - 1] + c->lhat[k]);", "c->Dh[k] = c->lhat[k];"),
    ("voronoi_B_right", "B on Voronoi domains from the right element only",
     "c->Bv[3 * k + q] = (2.0 * c->Dh[k]) / (c->lhat[k - 1] / c->B[3 * (k - 1) + q] + c->lhat[k] / c->B[3 * k + q]);",
     "c->Bv[3 * k + q] = c->B[3 * k + q];"),
    ("sigma_no_e", "sigma = Q t - e3 (unit tangent instead of r' = e t)",
     "= e[j] * Qt[", "= Qt["),
    ("dyn_sigma_no_e", "sigma = Q t - e3 in the dynamics",
     "for (int q = 0; q < 3; ++q) c->sig[3 * j + q] = c->e[j] * Qt[q] - e3[q];",
     "for (int q = 0; q < 3; ++q) c->sig[3 * j + q] = Qt[q] - e3[q];"),
    ("kappa_transposed", "kappa = logrot(Q_{k-1} Q_k^T)",
     "m_mul_t(Q + 9 * k, Q + 9 * (k - 1), R);", "m_mul_t(Q + 9 * (k - 1), Q + 9 * k, R);"),
    ("rot_sign", "rot(v) = exp(+[v]x)",
     "R[i] = ((i % 4) == 0 ? 1.0 : 0.0) - a * K[i] + b * K2[i];", "R[i] = ((i % 4) == 0 ? 1.0 : 0.0) + a * K[i] + b * K2[i];"),
    ("rot_b_sign", "rot(v) = I - a [v]x - b [v]x^2",
     "R[i] = ((i % 4) == 0 ? 1.0 : 0.0) - a * K[i] + b * K2[i];", "R[i] = ((i % 4) == 0 ? 1.0 : 0.0) - a * K[i] - b * K2[i];"),
    ("logrot_sign", "logrot returns +(theta / 2s) w",
     "v[0] = -f * w[0]; v[1] = -f * w[1]; v[2] = -f * w[2];", "v[0] = f * w[0]; v[1] = f * w[1]; v[2] = f * w[2];"),
    ("rotate_transposed", "Q <- Q rot(h w) (right multiplication)",
     "m_mul(R, Q + 9 * j, Q + 9 * j);", "m_mul(Q + 9 * j, R, Q + 9 * j);"),
    ("drift_full_step", "drift by h instead of h/2",
     "stage_drift(c, r, v, Q, w, 0.5 * h);", "stage_drift(c, r, v, Q, w, h);"),
    ("forcing_time_start", "time-dependent forcing at t_n instead of t_n + h/2",
     "double t_half = tt + 0.5 * dt;", "double t_half = tt;"),
    ("tip_at_start", "tip load on node 0 of a rod clamped at s = 0",
     "c->tip_node = (c->clamp == 1) ? 0 : N;", "c->tip_node = 0;"),
    ("bend_B_index", "B3 = G I1 instead of G (I1 + I2)",
     "c->B[3 * j + 2] = G * (I1 + I2);", "c->B[3 * j + 2] = G * I1;"),
    ("inertia_J3", "J3 = rho lhat I1 instead of rho lhat (I1 + I2)",
     "c->J[3 * j + 2] = rho * lh * (I1 + I2);", "c->J[3 * j + 2] = rho * lh * I1;"),
    ("shear_stiffness_no_alpha", "S1 = G A (no shear coefficient)",
     "c->S[3 * j + 0] = ac * G * A; c->S[3 * j + 1] = ac * G * A;", "c->S[3 * j + 0] = G * A; c->S[3 * j + 1] = G * A;"),
    ("bend_moment_difference_sign", "C = (m_j - m_{j+1}) + ...",
     "Cj[q] = (mn - mc) + 0.5 * (bn + bc);", "Cj[q] = (mc - mn) + 0.5 * (bn + bc);"),
    ("magnetic_cross_order", "c_mag = (Q b) x m instead of m x (Q b) (PAPER.md:266)",
     "v_cross(P->magnetization + 3 * (c->e0 + j), Qb, mb);", "v_cross(Qb, P->magnetization + 3 * (c->e0 + j), mb);"),
    ("magnetic_lab_field", "magnetic couple with the lab-frame b instead of Q b",
     "m_vec(Q + 9 * j, b, Qb);", "mt_vec(Q + 9 * j, b, Qb);"),
    ("muscle_pair_sign", "muscular couple pair with equal signs (not net-zero)",
     "if (j + 1 <= N - 1) Cj[P->musc_component] -= muscle_tau(P, rod, c, j + 1, t);",
     "if (j + 1 <= N - 1) Cj[P->musc_component] += muscle_tau(P, rod, c, j + 1, t);"),
    ("actuation_wave_direction", "rest-curvature wave sin(2 pi (s/L + f t))",
     "sin(2.0 * PI * (s / P->act_L[rod] - P->act_f[rod] * t))", "sin(2.0 * PI * (s / P->act_L[rod] + P->act_f[rod] * t))"),
    ("rest_kappa_sign", "m = B (kappa + kappa0) / eps^3",
     "c->mbar[3 * k + q] = c->Bv[3 * k + q] * (c->kap[3 * k + q] - k0[q]) / e3k;",
     "c->mbar[3 * k + q] = c->Bv[3 * k + q] * (c->kap[3 * k + q] + k0[q]) / e3k;"),
    ("gravity_weight_per_node", "gravity m g replaced by the element mass on every node",
     "f += c->m[i] * P->gravity[q];", "f += c->me[0] * P->gravity[q];"),
    ("clamp_rates_kept", "clamped element keeps its angular velocity",
     "if (c->clamp == 0) { memset(v, 0, 3 * sizeof(double)); memset(w, 0, 3 * sizeof(double)); }",
     "if (c->clamp == 0) { memset(v, 0, 3 * sizeof(double)); }"),
    ("n_not_rotated", "n = nbar (local frame used as lab)",
     "mt_vec(Q + 9 * j, c->nbar + 3 * j, c->nlab + 3 * j);", "m_vec(Q + 9 * j, c->nbar + 3 * j, c->nlab + 3 * j);"),
]


# Where each mutant was first seen to die (a run-order hint only: the hinted tests run first, and if
# they all pass the whole suite runs, so a stale hint can only cost time, never hide a survivor).
HINTS = {
    "drift_full_step": "test_oracle_dynamics.py::test_free_drift",
    "rotate_transposed": "test_oracle_dynamics.py::test_rigid_spin_about_axis",
    "forcing_time_start": "test_oracle_contact.py::test_coulomb_sliding_deceleration",
    "tip_at_start": "test_oracle_dynamics.py::test_cantilever_cfg1",
    "clamp_rates_kept": "test_oracle_dynamics.py::test_clamps_hold_exactly",
    "magnetic_cross_order": "test_oracle_magnetic.py::test_couple_is_lhat_m_cross_Qb",
    "magnetic_lab_field": "test_oracle_magnetic.py::test_couple_equals_rotated_lab_dipole_torque",
    "muscle_pair_sign": "test_oracle_muscle.py::test_net_zero_and_pattern",
    "actuation_wave_direction": "test_oracle_dynamics.py::test_actuation_wave_travels_toward_tip",
    "shear_torque_sign": "test_oracle_contact.py::test_rest_on_floor_reaction_equals_weight",
}


def tests_order():
    """The new finite-strain pins first (fast), then the rest of the oracle suite."""
    tdir = os.path.join(ROOT, "tests")
    files = sorted(f for f in os.listdir(tdir) if f.startswith("test_oracle_") and f.endswith(".py")
                   and f != "test_oracle_mutants.py")
    for first in reversed(("test_oracle_finite_strain.py", "test_oracle_loads.py", "test_oracle_strains.py",
                           "test_oracle_so3.py")):
        if first in files:
            files.remove(first)
            files.insert(0, first)
    return [os.path.join(tdir, f) for f in files]


def run_mutant(name, old, new, src_text, workdir):
    import oracle
    if old not in src_text:
        return "unapplicable", f"text not found: {old[:60]}"
    mdir = os.path.join(workdir, name)
    os.makedirs(mdir, exist_ok=True)
    src = os.path.join(mdir, "oracle.c")
    with open(src, "w") as f:
        f.write(src_text.replace(old, new))
    with open(os.path.join(mdir, "oracle.h"), "w") as f:
        f.write(open(os.path.join(ROOT, "oracle", "oracle.h")).read())
    try:
        lib = oracle.build(force=True, src=src, out=os.path.join(mdir, "liboracle.so"))
    except subprocess.CalledProcessError as exc:
        return "error", f"build failed: {exc}"
    env = dict(os.environ, ER_ORACLE_LIB=lib, PYTHONDONTWRITEBYTECODE="1")
    base = [sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", "-m", "not gpu"]
    p = None
    if name in HINTS:
        p = subprocess.run(base + [os.path.join(ROOT, "tests", HINTS[name])], cwd=ROOT, env=env,
                           capture_output=True, text=True)
        if p.returncode == 0:
            p = None
    if p is None:
        p = subprocess.run(base + tests_order(), cwd=ROOT, env=env, capture_output=True, text=True)
    failed = [ln.split(" ")[1] for ln in p.stdout.splitlines() if ln.startswith("FAILED ")]
    if p.returncode == 0:
        return "SURVIVED", ""
    if p.returncode == 1 and failed:
        return "killed", failed[0]
    return "error", p.stdout[-800:] + p.stderr[-800:]


def main(argv):
    want = set(argv)
    src_text = open(os.path.join(ROOT, "oracle", "oracle.c")).read()
    from concurrent.futures import ThreadPoolExecutor
    jobs = [m for m in MUTANTS if not want or m[0] in want]
    n_par = max(1, min(len(jobs), int(os.environ.get("ER_MUTANT_JOBS", "0")) or
                       len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else 4))
    rows, bad = [], []
    with tempfile.TemporaryDirectory(prefix="oracle_mutants_") as wd:
        def one(m):
            name, what, old, new = m
            t0 = time.time()
            verdict, info = run_mutant(name, old, new, src_text, wd)
            print(f"{name:28s} {verdict:12s} {time.time() - t0:6.1f}s  {what}  [{info.strip()[:200]}]", flush=True)
            return name, verdict
        with ThreadPoolExecutor(n_par) as ex:
            for name, verdict in ex.map(one, jobs):
                rows.append(name)
                if verdict != "killed":
                    bad.append(name)
    print(f"{len(rows) - len(bad)}/{len(rows)} mutants killed" + (f"; NOT killed: {bad}" if bad else ""))
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
