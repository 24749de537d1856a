"""Generate golden fixtures by running the UNMODIFIED reference solver.

Run in the build container (``/root/reference`` is not on the GPU box):

    python tests/golden/make_golden.py

It imports ``conic_ipm`` from ``/root/reference/pkg/src`` and writes

* ``tests/golden/instances/<name>.json`` — problem data, settings, the
  reference SolveResult and its per-iteration trace (μ, α_a, σ, α_c, τ, κ)
  captured through the reference's ``observer`` seam (``ipm.py:475-480``);
* ``tests/golden/kernels.json`` — kernel-level known answers: scaling
  updates, combined_ds, apply_H, step lengths, neighbourhood tests,
  conjugate points, batched SOC residuals (SPEC AC11) and LDL examples.

The fixtures pin the oracle (``oracle/``) and the CUDA path.
"""
from __future__ import annotations

import json
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402

import conic_ipm as ref  # noqa: E402
from conic_ipm.cones import barriers as rbar  # noqa: E402
from conic_ipm.cones import scaling as rsc  # noqa: E402
from conic_ipm.cones import steps as rst  # noqa: E402
from conic_ipm.kkt import system as rsys  # noqa: E402

from paper_2412_19027_b200 import generators as G  # noqa: E402


def flist(a):
    return [float(v) for v in np.asarray(a, dtype=np.float64).ravel()]


def csr_doc(m):
    return {"nrows": int(m.nrows), "ncols": int(m.ncols), "rowptr": [int(v) for v in m.rowptr],
            "colidx": [int(v) for v in m.colidx], "values": flist(m.values)}


def cone_doc(c):
    d = {"kind": c.kind, "dim": int(c.dim)}
    if c.alpha is not None:
        d["alpha"] = float(c.alpha)
    if c.side is not None:
        d["side"] = int(c.side)
    return d


def to_ref(p):
    conv = {"zero": lambda c: ref.zero_cone(c.dim), "nonneg": lambda c: ref.nonneg_cone(c.dim),
            "soc": lambda c: ref.soc_cone(c.dim), "exp": lambda c: ref.exp_cone(),
            "pow": lambda c: ref.pow_cone(c.alpha), "psd": lambda c: ref.psd_cone(c.side)}
    P = ref.CsrMatrix(p.P.nrows, p.P.ncols, p.P.rowptr, p.P.colidx, p.P.values)
    A = ref.CsrMatrix(p.A.nrows, p.A.ncols, p.A.rowptr, p.A.colidx, p.A.values)
    return ref.ProblemData(P, A, p.q, p.b, [conv[c.kind](c) for c in p.cones])


def run_instance(name, prob, eps=1e-8, precision="full", max_iter=200):
    trace = []

    def obs(d):
        st = d["state"]
        trace.append({"it": d["iteration"], "mu": st.mu, "tau": st.tau, "kappa": st.kappa,
                      "alpha_affine": d["alpha_affine"], "sigma": d["sigma"],
                      "alpha_combined": d["alpha_combined"]})

    settings = ref.SolverSettings(eps_feas=eps, precision=precision, max_iter=max_iter)
    solver = ref.Solver(prob, settings)
    res = solver.solve(observer=obs)
    doc = {
        "name": name,
        "problem": {"P": csr_doc(prob.P), "A": csr_doc(prob.A), "q": flist(prob.q),
                    "b": flist(prob.b), "cones": [cone_doc(c) for c in prob.cones]},
        "settings": {"eps_feas": eps, "precision": precision, "max_iter": max_iter},
        "result": {"status": res.status, "iterations": res.iterations,
                   "obj_primal": res.obj_primal, "obj_dual": res.obj_dual,
                   "norm_rp": res.norm_rp, "norm_rd": res.norm_rd, "gap": res.gap,
                   "tau": res.tau, "kappa": res.kappa, "mu_initial": res.mu_initial,
                   "mu_final": res.mu_final, "x": flist(res.x), "z": flist(res.z),
                   "s": flist(res.s),
                   "certificate": None if res.certificate is None else flist(res.certificate)},
        "trace": trace,
        "kkt": {"num_symbolic": solver.kkt.num_symbolic, "num_numeric": solver.kkt.num_numeric},
    }
    print(f"{name:32s} {res.status:22s} it={res.iterations:3d} obj={res.obj_primal:.10g}")
    return doc


def instances():
    out = []
    for prec in ("full", "mixed"):
        sfx = "" if prec == "full" else "_mixed"
        out.append((f"lp_20x40{sfx}", G.gen_lp(20, 40, seed=1), 1e-8, prec))
        out.append((f"lasso_10x40{sfx}", G.gen_lasso(10, 40, seed=1), 1e-8, prec))
        out.append((f"mpc_s0{sfx}", G.gen_mpc(0), 1e-8, prec))
    out.append(("lp_60x120", G.gen_lp(60, 120, seed=2), 1e-8, "full"))
    out.append(("lp_150x300", G.gen_lp(150, 300, seed=3), 1e-8, "full"))
    out.append(("lasso_40x160", G.gen_lasso(40, 160, seed=2), 1e-8, "full"))
    out.append(("socp_10", G.gen_socp(10, seed=1), 1e-8, "full"))
    out.append(("socp_40", G.gen_socp(40, seed=2), 1e-8, "full"))
    out.append(("exppow_20_8", G.gen_exppow(20, 8, seed=1, block=10), 1e-8, "full"))
    out.append(("exppow_40_16", G.gen_exppow(40, 16, seed=2, block=10), 1e-6, "full"))
    out.append(("exp_only_30", G.gen_exppow(30, 0, seed=3, block=10), 1e-6, "full"))
    out.append(("psd_4x3", G.gen_psd(4, 3, seed=1), 1e-8, "full"))
    out.append(("psd_6x4", G.gen_psd(6, 4, seed=2), 1e-8, "full"))
    out.append(("psd_3x6", G.gen_psd(3, 6, seed=3), 1e-8, "full"))
    out.append(("mpc_s1", G.gen_mpc(1), 1e-8, "full"))
    return out


def ref_family_instances():
    """Instances from the reference's own generators (converted to dicts)."""
    out = []
    out.append(("ref_portfolio_20", ref.gen_portfolio(20, seed=3), 1e-8))
    out.append(("ref_portfolio_sym", ref.gen_portfolio(2, mu=np.zeros(2), factor=np.zeros((2, 1)),
                                                       dvec=np.ones(2)), 1e-8))
    out.append(("ref_huber_8", ref.gen_huber(8, seed=2), 1e-8))
    for n in (4, 16):
        out.append((f"ref_entropy_simplex_{n}", ref.gen_entropy(n, seed=0, include_ineq=False), 1e-6))
    out.append(("ref_entropy_12", ref.gen_entropy(12, seed=1), 1e-6))
    out.append(("ref_multistage_24_3_2", ref.gen_multistage_portfolio(24, 3, 2, seed=4), 1e-8))
    # min ½x² s.t. x >= 1
    P = ref.CsrMatrix.from_dense([[1.0]])
    A = ref.CsrMatrix.from_dense([[-1.0]])
    out.append(("halfx2_x_ge_1", ref.ProblemData(P, A, np.zeros(1), np.array([-1.0]),
                                                  [ref.nonneg_cone(1)]), 1e-8))
    # primal infeasible: x >= 0, x <= -1
    P = ref.CsrMatrix.zeros(1, 1)
    A = ref.CsrMatrix.from_dense([[-1.0], [1.0]])
    out.append(("primal_infeasible_lp", ref.ProblemData(P, A, np.array([1.0]), np.array([0.0, -1.0]),
                                                         [ref.nonneg_cone(2)]), 1e-8))
    # dual infeasible (unbounded): min -x s.t. x >= 0  (reference ends insufficient_progress)
    P = ref.CsrMatrix.zeros(1, 1)
    A = ref.CsrMatrix.from_dense([[-1.0]])
    out.append(("dual_infeasible_lp", ref.ProblemData(P, A, np.array([-1.0]), np.array([0.0]),
                                                       [ref.nonneg_cone(1)]), 1e-8))
    # unbounded 2-var LP with a free direction: min -x1 s.t. x2 = 0, x1 >= 0
    P = ref.CsrMatrix.zeros(2, 2)
    A = ref.CsrMatrix.from_dense([[0.0, 1.0], [-1.0, 0.0]])
    out.append(("dual_infeasible_lp2", ref.ProblemData(P, A, np.array([-1.0, 0.0]), np.zeros(2),
                                                        [ref.zero_cone(1), ref.nonneg_cone(1)]), 1e-8))
    return out


# ---------------------------------------------------------------------------
# kernel-level fixtures
# ---------------------------------------------------------------------------

def interior_pair(rng, cones):
    """Random strictly interior (s, z) for a ConeSet (reference conventions)."""
    s = np.zeros(cones.m)
    z = np.zeros(cones.m)
    nn0, nnd = cones.nonneg_start, cones.nonneg_dim
    s[nn0:nn0 + nnd] = rng.uniform(0.1, 3.0, nnd)
    z[nn0:nn0 + nnd] = rng.uniform(0.1, 3.0, nnd)
    for off, dim in cones.socs:
        for v in (s, z):
            u = rng.standard_normal(dim - 1)
            v[off:off + dim] = np.concatenate([[np.linalg.norm(u) + rng.uniform(0.1, 2.0)], u])
    for off in cones.exps:
        # primal: (x, y, z) with y exp(x/y) < z ; dual: (u, v, w) with u<0, -u exp(v/u) < e w
        y = rng.uniform(0.5, 2.0)
        x = rng.uniform(-2.0, 1.0)
        zz = y * np.exp(x / y) * rng.uniform(1.2, 3.0)
        s[off:off + 3] = (x, y, zz)
        u = -rng.uniform(0.5, 2.0)
        vv = rng.uniform(-1.0, 2.0)
        w = -u * np.exp(vv / u) / np.e * rng.uniform(1.2, 3.0)
        z[off:off + 3] = (u, vv, w)
    for off, a in cones.pows:
        x, y = rng.uniform(0.5, 2.0, 2)
        bound = x ** a * y ** (1 - a)
        s[off:off + 3] = (x, y, bound * rng.uniform(-0.8, 0.8))
        u, vv = rng.uniform(0.5, 2.0, 2)
        bd = (u / a) ** a * (vv / (1 - a)) ** (1 - a)
        z[off:off + 3] = (u, vv, bd * rng.uniform(-0.8, 0.8))
    for off, side in cones.psds:
        from conic_ipm.cones.psdcone import svec, triangle_dim
        d = triangle_dim(side)
        for v in (s, z):
            g = rng.standard_normal((side, side))
            v[off:off + d] = svec(g @ g.T / side + 0.5 * np.eye(side))
    return s, z


def scaling_doc(sc, cones):
    diag, blocks = sc.kkt_values()
    return {"diag": flist(diag), "blocks": [[int(off), flist(b)] for off, b in blocks],
            "nn_w": flist(sc.nn_w), "nn_lam": flist(sc.nn_lam),
            "soc": [{"w": flist(x.w), "eta": float(x.eta), "lam": flist(x.lam)} for x in sc.socs],
            "nsym": [{"h": flist(x.h), "grad": flist(x.grad_z), "hess": flist(x.hess_z),
                      "zt": flist(x.z_tilde), "mu_c": x.mu_cone, "mu_t": x.mu_tilde} for x in sc.nsyms],
            "psd_lam": [flist(np.sort(x.lam)) for x in sc.psds]}


def kernel_fixtures():
    rng = np.random.default_rng(2024)
    cases = []
    specs = [
        [ref.zero_cone(3), ref.nonneg_cone(7)],
        [ref.nonneg_cone(4), ref.soc_cone(3), ref.soc_cone(5), ref.soc_cone(2)],
        [ref.exp_cone(), ref.exp_cone(), ref.exp_cone()],
        [ref.pow_cone(0.3), ref.pow_cone(0.5), ref.pow_cone(0.75)],
        [ref.psd_cone(2), ref.psd_cone(3)],
        [ref.zero_cone(2), ref.nonneg_cone(3), ref.soc_cone(4), ref.exp_cone(), ref.pow_cone(0.4),
         ref.psd_cone(3)],
    ]
    for ci, spec in enumerate(specs):
        cones = ref.ConeSet.from_specs(spec)
        for rep in range(4):
            s, z = interior_pair(rng, cones)
            mu = float(s @ z) / max(1, cones.degree)
            try:
                sc = rsc.update_scaling(cones, s, z, mu)
            except ref.ConicError as e:  # pragma: no cover - fixture generation
                print("skip", ci, rep, e)
                continue
            v = rng.standard_normal(cones.m)
            v[:cones.zero_dim] = 0.0
            dz = rng.standard_normal(cones.m) * 0.3
            ds = rng.standard_normal(cones.m) * 0.3
            ds[:cones.zero_dim] = 0.0
            sigma = float(rng.uniform(0.0, 1.0))
            hv = rsc.apply_H(sc, v)
            try:
                cds = rsc.combined_ds(sc, cones, s, z, dz, ds, sigma, mu)
            except ref.ConicError:
                cds = None
            req = rst.StepLengthRequest(z=z, s=s, dz=dz, ds=ds, tau=1.0, kappa=1.0,
                                        dtau=-0.5, dkappa=0.2)
            try:
                alpha = rst.step_length(req, cones)
            except ref.ConicError:
                alpha = None
            nb = {str(beta): bool(rsc.neighborhood_ok(cones, s, z, mu, beta)) for beta in (1e-6, 0.5, 0.9)}
            cases.append({
                "cones": [cone_doc(c) for c in spec], "s": flist(s), "z": flist(z), "mu": mu,
                "scaling": scaling_doc(sc, cones), "v": flist(v), "Hv": flist(hv),
                "dz": flist(dz), "ds": flist(ds), "sigma": sigma,
                "combined_ds": None if cds is None else flist(cds),
                "step": {"tau": 1.0, "kappa": 1.0, "dtau": -0.5, "dkappa": 0.2, "alpha": alpha},
                "neighborhood": nb,
                "in_cone": bool(ref.is_in_cone(cones, s, strict=True)),
                "in_dual": bool(ref.is_in_dual_cone(cones, z, strict=True)),
            })
    # conjugate points of exp / pow
    conj = []
    for _ in range(40):
        y = rng.uniform(0.2, 3.0)
        x = rng.uniform(-3.0, 2.0)
        zz = y * np.exp(x / y) * rng.uniform(1.01, 5.0)
        s = np.array([x, y, zz])
        conj.append({"kind": "exp", "s": flist(s), "w": flist(rbar.exp_conjugate_dual_point(s))})
    for _ in range(40):
        a = rng.uniform(0.1, 0.9)
        x, y = rng.uniform(0.2, 3.0, 2)
        bd = x ** a * y ** (1 - a)
        s = np.array([x, y, bd * rng.uniform(-0.99, 0.99)])
        conj.append({"kind": "pow", "alpha": a, "s": flist(s),
                     "w": flist(rbar.pow_conjugate_dual_point(s, a))})
    # batched SOC residuals (SPEC AC11)
    dims = [5, 3, 2, 9, 17, 33, 64, 100, 2]
    cs = ref.ConeSet.from_specs([ref.soc_cone(d) for d in dims])
    xv = rng.standard_normal(cs.m)
    xv[0:5] = (5, 3, 4, 0, 0)
    soc_res = {"dims": dims, "x": flist(xv), "r": flist(rst.soc_residuals_batch(cs, xv))}
    # LDL examples: K=[[4,2],[2,-2]] -> D=(4,-3)
    ldl = []
    for kmat, n in (([[4.0, 2.0], [2.0, -2.0]], 1), ([[2.0, 0.0], [0.0, -3.0]], 1)):
        kd = np.array(kmat)
        P = ref.CsrMatrix.from_dense(kd[:n, :n])
        A = ref.CsrMatrix.from_dense(kd[n:, :n])
        cones = ref.ConeSet.from_specs([ref.nonneg_cone(kd.shape[0] - n)])
        sysk = rsys.assemble(P, A, cones, delta_s=0.0, delta_d=0.0)
        sysk.set_scaling(np.array([-kd[n, n]]), [])
        sysk.numeric_factor()
        dvec = sysk._d[np.float64][sysk.iperm]
        b = np.array([1.0, 2.0])
        sol = sysk.solve_refined(b)
        ldl.append({"K": flist(kd), "n": n, "D_in_original_order": flist(dvec), "b": flist(b),
                    "x": flist(sol.x), "steps": sol.steps})
    return {"cones": cases, "conjugate": conj, "soc_residuals": soc_res, "ldl": ldl}


def main():
    os.makedirs(os.path.join(HERE, "instances"), exist_ok=True)
    for name, prob, eps, prec in instances():
        doc = run_instance(name, to_ref(prob), eps=eps, precision=prec)
        with open(os.path.join(HERE, "instances", name + ".json"), "w") as f:
            json.dump(doc, f)
    for name, prob, eps in ref_family_instances():
        doc = run_instance(name, prob, eps=eps)
        with open(os.path.join(HERE, "instances", name + ".json"), "w") as f:
            json.dump(doc, f)
    with open(os.path.join(HERE, "kernels.json"), "w") as f:
        json.dump(kernel_fixtures(), f)
    print("wrote fixtures to", HERE)


if __name__ == "__main__":
    main()
