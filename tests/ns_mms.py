"""TEST INFRASTRUCTURE — exact right-hand side of the reacting Navier-Stokes
equations for a manufactured smooth periodic state, by symbolic calculus
(sympy), independent of the oracle's and the kernels' discretisation.

Equations:
  d rho/dt     = -div(rho u)
  d rho u/dt   = -div(rho u u) - grad p + div tau
  d rho Y_k/dt = -div(rho Y_k u) + rho omega_k - div F_k
  d rho E/dt   = -div[(rho E + p) u] + div(lambda grad T) + div(tau . u)
                 - div sum_k F_k h_k
  tau_ij = eta (d_j u_i + d_i u_j - 2/3 delta_ij div u) + xi delta_ij div u
  Fbar_k = -rho D_k (grad X_k + (X_k - Y_k) grad p / p)
  V_c = sum_l Fbar_l,  F_k = Fbar_k - Y_k V_c
with the ideal-gas mixture EOS and the synthetic models of
include/smc_mechanism.h (the input deck is parsed from that header, so the
data are the ones the kernels and the oracle use; the algebra here is not).

Each physical term is returned separately, matching the oracle's term mask
(oracle/ns_oracle.h OR_T_*): HYP, VISC, HEAT, SPEC, ENTH, CHEM.  The state is
given on the node grid x_i = i dx of the periodic box [0, L)^3.
"""
from __future__ import annotations

import functools
import os
import re

import numpy as np
import sympy as sp

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "smc_mechanism.h")

HYP, VISC, HEAT, SPEC, ENTH, CHEM = 1, 2, 4, 8, 16, 32
TERMS = {"hyp": HYP, "visc": VISC, "heat": HEAT, "spec": SPEC, "enth": ENTH, "chem": CHEM}
L_BOX = 3.2e-3  # m: dx = 1e-4 m at n = 32, the configs' spacing


def _nums(text):
    return [float(v) for v in re.findall(r"[-+]?\d+\.?\d*(?:[eE][-+]?\d+)?", text)]


@functools.lru_cache(maxsize=1)
def mechanism() -> dict:
    """The input deck of smc_mechanism.h as Python numbers."""
    h = open(HEADER).read()
    scal = {k: float(v) for k, v in re.findall(r"#define SMC_(RU|T_REF|TRANSPORT_EXP|XI_OVER_ETA)"
                                                 r"\s+([-+\d.eE]+)", h)}

    def arr(name):
        body = re.search(name + r"[^=]*=\s*\{(.*?)\};", h, re.S).group(1)
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        return _nums(body)

    sp_names = re.search(r"enum \{(.*?)\};", h, re.S).group(1)
    idx = {nm.strip(): i for i, nm in enumerate(sp_names.replace("= 0", "").split(","))}
    rx = []
    lst = h[h.index("#define SMC_REACTION_LIST"):h.index("#define SMC_REACTION_ENTRY")]
    for args in re.findall(r"X\(([^)]*)\)", lst):
        parts = [a.strip() for a in args.split(",")]
        if parts[0] == "reactant0..2":  # the macro's own documentation line
            continue
        sp_of = [idx[a] if a in idx else int(a) for a in parts[:6]]
        rx.append(dict(reac=[i for i in sp_of[:3] if i >= 0], prod=[i for i in sp_of[3:6] if i >= 0],
                       tb=int(parts[6]), fwd=[float(v) for v in parts[7:10]],
                       rev=[float(v) for v in parts[10:13]]))
    thermo = np.array(arr("SMC_THERMO")).reshape(9, 4)
    return dict(W=arr("SMC_W"), thermo=thermo, mu0=arr("SMC_MU0"), lam0=arr("SMC_LAM0"),
                rhoD0=arr("SMC_RHOD0"), reactions=rx, Ru=scal["RU"], Tref=scal["T_REF"],
                texp=scal["TRANSPORT_EXP"], xi=scal["XI_OVER_ETA"])


X_, Y_, Z_ = sp.symbols("x y z", real=True)


def primitive_fields(kind: str = "mixed"):
    """Manufactured primitives (T, p, (u, v, w), Y_0..8) as sympy expressions
    of x, y, z, periodic on [0, L)^3; every term of the RHS is active and
    every mixed derivative is nonzero."""
    k = 2 * sp.pi / L_BOX
    x, y, z = X_, Y_, Z_
    T = 1200 + 150 * sp.sin(k * x + 0.3) * sp.cos(k * y - 0.2) + 120 * sp.sin(k * z + 0.5)
    if kind == "hot":  # reactive: T up to ~1750 K so the chemistry is fast
        T = T + 250 * sp.cos(k * x) * sp.cos(k * y) * sp.cos(k * z) + 120
    p = 101325 * (1 + 0.03 * sp.cos(k * x + k * z + 0.1) + 0.02 * sp.sin(k * y))
    u = [10 * sp.sin(k * x + 0.1) * sp.cos(k * y) + 4 * sp.sin(k * z - 0.4),
         8 * sp.cos(k * x - 0.3) * sp.sin(k * z + 0.2) + 3 * sp.cos(k * y),
         6 * sp.sin(k * y + 0.7) * sp.cos(k * x) - 5 * sp.cos(k * z + 0.1)]
    Y = [0.02 + 0.006 * sp.sin(k * x) * sp.cos(k * z + 0.2),           # H2
         0.22 + 0.02 * sp.cos(k * y + 0.4) * sp.sin(k * x - 0.1),      # O2
         0.02 + 0.008 * sp.sin(k * z + k * y),                          # H2O
         2e-4 + 1e-4 * sp.cos(k * x - k * z),                           # H
         3e-4 + 1e-4 * sp.sin(k * y - 0.3),                             # O
         1e-3 + 5e-4 * sp.cos(k * z + 0.6) * sp.cos(k * x),             # OH
         1e-4 + 5e-5 * sp.sin(k * x + k * y),                           # HO2
         5e-5 + 2e-5 * sp.cos(k * y - k * z)]                           # H2O2
    Y.append(1 - sum(Y))                                                # N2
    return T, p, u, Y


def _div(vec):
    return sum(sp.diff(vec[j], v) for j, v in enumerate((X_, Y_, Z_)))


def _grad(f):
    return [sp.diff(f, v) for v in (X_, Y_, Z_)]


@functools.lru_cache(maxsize=4)
def exact_rhs(kind: str = "mixed"):
    """Lambdified exact terms: f(x, y, z) -> dict term -> list of 14 arrays,
    plus the conserved state and the primitives."""
    m = mechanism()
    T, p, u, Y = primitive_fields(kind)
    W, th, Ru = m["W"], m["thermo"], m["Ru"]
    nsp = len(W)
    Rk = [Ru / W[k] for k in range(nsp)]
    h = [Rk[k] * (th[k][0] * T + th[k][1] * T ** 2 / 2 + th[k][2] * T ** 3 / 3 + th[k][3])
         for k in range(nsp)]
    e_k = [h[k] - Rk[k] * T for k in range(nsp)]
    Wmix = 1 / sum(Y[k] / W[k] for k in range(nsp))
    X = [Y[k] * Wmix / W[k] for k in range(nsp)]
    rho = p * Wmix / (Ru * T)
    e = sum(Y[k] * e_k[k] for k in range(nsp))
    E = e + (u[0] ** 2 + u[1] ** 2 + u[2] ** 2) / 2
    s = (T / m["Tref"]) ** m["texp"]
    eta = s * sum(X[k] * m["mu0"][k] for k in range(nsp))
    lam = s * sum(X[k] * m["lam0"][k] for k in range(nsp))
    xi = m["xi"] * eta
    rhoD = [m["rhoD0"][k] * s for k in range(nsp)]
    gu = [_grad(ui) for ui in u]  # gu[i][j] = d_j u_i
    divu = gu[0][0] + gu[1][1] + gu[2][2]
    tau = [[eta * (gu[i][j] + gu[j][i]) + (xi - sp.Rational(2, 3) * eta) * divu * int(i == j)
            for j in range(3)] for i in range(3)]
    gp = _grad(p)
    Fbar = [[-rhoD[k] * (sp.diff(X[k], v) + (X[k] - Y[k]) * gp[j] / p)
             for j, v in enumerate((X_, Y_, Z_))] for k in range(nsp)]
    Vc = [sum(Fbar[k][j] for k in range(nsp)) for j in range(3)]
    F = [[Fbar[k][j] - Y[k] * Vc[j] for j in range(3)] for k in range(nsp)]
    zero = sp.Integer(0)
    terms = {}
    # HYP
    hyp = [-_div([rho * u[j] for j in range(3)])]
    hyp += [-_div([rho * u[i] * u[j] + p * int(i == j) for j in range(3)]) for i in range(3)]
    hyp += [-_div([(rho * E + p) * u[j] for j in range(3)])]
    hyp += [-_div([rho * Y[k] * u[j] for j in range(3)]) for k in range(nsp)]
    terms["hyp"] = hyp
    # VISC
    visc = [zero] + [_div(tau[i]) for i in range(3)]
    visc += [_div([sum(tau[i][j] * u[i] for i in range(3)) for j in range(3)])]
    terms["visc"] = visc + [zero] * nsp
    # HEAT
    terms["heat"] = [zero] * 4 + [_div([lam * sp.diff(T, v) for v in (X_, Y_, Z_)])] + [zero] * nsp
    # SPEC
    terms["spec"] = [zero] * 5 + [-_div(F[k]) for k in range(nsp)]
    # ENTH
    terms["enth"] = [zero] * 4 + [-_div([sum(F[k][j] * h[k] for k in range(nsp))
                                         for j in range(3)])] + [zero] * nsp
    # CHEM: rho omega_k W_k, forward and reverse rates independent
    Cc = [rho * Y[k] / W[k] for k in range(nsp)]
    Mtb = sum(Cc)
    om = [zero] * nsp
    for r in m["reactions"]:
        kf = r["fwd"][0] * T ** r["fwd"][1] * sp.exp(-r["fwd"][2] / (Ru * T))
        kr = r["rev"][0] * T ** r["rev"][1] * sp.exp(-r["rev"][2] / (Ru * T))
        qf, qr = kf, kr
        for i in r["reac"]:
            qf = qf * Cc[i]
        for i in r["prod"]:
            qr = qr * Cc[i]
        if r["tb"]:
            qf, qr = qf * Mtb, qr * Mtb
        q = qf - qr
        for i in r["reac"]:
            om[i] = om[i] - q
        for i in r["prod"]:
            om[i] = om[i] + q
    terms["chem"] = [zero] * 5 + [W[k] * om[k] for k in range(nsp)]
    cons = [rho] + [rho * ui for ui in u] + [rho * E] + [rho * Y[k] for k in range(nsp)]
    names = list(terms)
    flat = [ex for nm in names for ex in terms[nm]] + cons
    f = sp.lambdify((X_, Y_, Z_), flat, modules="numpy", cse=True)
    return f, names


def grid(n: int):
    g = np.arange(n) * (L_BOX / n)
    z, y, x = np.meshgrid(g, g, g, indexing="ij")  # (z, y, x): x fastest
    return x, y, z


def evaluate(n: int, kind: str = "mixed"):
    """(U, {term: exact (14, n, n, n)}, dx) on the n^3 node grid."""
    f, names = exact_rhs(kind)
    x, y, z = grid(n)
    vals = f(x, y, z)
    shape = (n, n, n)
    full = [np.broadcast_to(np.asarray(v, dtype=np.float64), shape) for v in vals]
    out = {}
    for i, nm in enumerate(names):
        out[nm] = np.ascontiguousarray(np.stack(full[14 * i:14 * (i + 1)]))
    U = np.ascontiguousarray(np.stack(full[14 * len(names):]))
    return U, out, L_BOX / n


def term_error(num: np.ndarray, exact: np.ndarray) -> float:
    """max over the nonzero components of max |num - exact| / max |exact|."""
    errs = [np.abs(num[v] - exact[v]).max() / np.abs(exact[v]).max()
            for v in range(exact.shape[0]) if np.abs(exact[v]).max() > 0]
    return float(max(errs))
