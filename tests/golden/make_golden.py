"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Run in the build container (needs /root/reference and oracle/_ref, built by
oracle/build_ref.sh):

    python tests/golden/make_golden.py

Every case stores the raw inputs (observation arrays + COO triplets in
original row order, optional strata) and what the compiled reference module
(`_survscan`, bindings/survscan_py.cpp) returns for them:
  * per-column (gradient, hessian) at a probe beta  (survscan_py.cpp:287-319)
  * log-likelihood at the probe beta and at zero
  * full fits (beta, objective, cycles, trace) under several penalties
Stratified cases have no reference counterpart: their expected
values are the composition sum of the reference run on each stratum's rows
(SURVEY.md §8c), and the stratified fit is a host CCD loop over those
per-stratum reference derivatives using the pinned oracle coordinate_step.
The fixtures are small (a few hundred KB total) and committed; the GPU box
never reads /root/reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
sys.path.insert(0, ROOT)
import _survscan as ref  # noqa: E402  (the reference module, oracle/_ref)

from oracle import oracle as orc  # noqa: E402


def raw_case(n, p, density, seed, *, valued=False, quant=None, cens=0.3,
             competing=0.0, dense_cols=0, scale=0.5):
    rng = np.random.default_rng(seed)
    mask = rng.random((n, p)) < density
    for j in range(min(dense_cols, p)):
        mask[:, j] = rng.random(n) < 0.6
    X = mask.astype(np.float64)
    if valued:
        X = np.where(mask, np.round(rng.normal(size=(n, p)), 3), 0.0)
        X[X == 0.0] = 0.0
    bt = rng.normal(size=p) * (rng.random(p) < 0.6) * scale
    eta = X @ bt
    t = rng.exponential(1.0 / np.exp(eta))
    status = np.ones(n, dtype=np.int64)
    if competing > 0:
        comp = rng.random(n) < competing
        status[comp] = 2
    if cens > 0:
        c = rng.exponential(np.quantile(t, 0.7) / max(cens, 1e-9), size=n)
        cz = c < t
        t = np.where(cz, c, t)
        status[cz] = 0
    if quant is not None:
        t = np.ceil(t * quant) / quant
    rows, cols = np.nonzero(X)
    return dict(times=t, status=status, rows=rows.astype(np.int64),
                cols=cols.astype(np.int64), values=X[rows, cols], n_cols=p)


def ref_dataset(c, subset=None):
    t, s = c["times"], c["status"]
    rows, cols, vals = c["rows"], c["cols"], c["values"]
    if subset is not None:
        remap = -np.ones(len(t), dtype=np.int64)
        remap[subset] = np.arange(len(subset))
        keep = remap[rows] >= 0
        rows, cols, vals = remap[rows[keep]], cols[keep], vals[keep]
        t, s = t[subset], s[subset]
    return ref.dataset_from_coo(t, s, rows, cols, vals, c["n_cols"])


def from_ref_sim(ds):
    """Extract a reference-simulated dataset (already sorted) as raw COO."""
    n, p = ds.n, ds.p
    X = np.array([[ds.covariate(i, j) for j in range(p)] for i in range(n)])
    rows, cols = np.nonzero(X)
    return dict(times=np.asarray(ds.times), status=np.asarray(ds.status).astype(np.int64),
                rows=rows.astype(np.int64), cols=cols.astype(np.int64),
                values=X[rows, cols], n_cols=p)


FITS = [("none", 0.0), ("l1", 0.5), ("l2", 2.0), ("l1", 25.0)]


def evaluate(name, c, model, beta_seed=7, beta_scale=0.3, fits=FITS, max_cycles=1000,
             extra=None):
    p = c["n_cols"]
    rng = np.random.default_rng(beta_seed)
    beta = rng.uniform(-beta_scale, beta_scale, size=p)
    ds = ref_dataset(c)
    out = dict(c)
    out.update(model=model, beta_probe=beta)
    gh = np.array([ref.grad_hessian(ds, model, beta, j, threads=1) for j in range(p)])
    gh0 = np.array([ref.grad_hessian(ds, model, np.zeros(p), j, threads=1) for j in range(p)])
    out["grad"], out["hess"] = gh[:, 0], gh[:, 1]
    out["grad0"], out["hess0"] = gh0[:, 0], gh0[:, 1]
    out["ll"] = ref.log_likelihood(ds, model, beta, threads=1)
    out["ll0"] = ref.log_likelihood(ds, model, np.zeros(p), threads=1)
    fit_names = []
    for k, (pen, lam) in enumerate(fits):
        r = ref.fit(ds, model=model, penalty=pen, strength=lam, max_cycles=max_cycles,
                    threads=1)
        key = f"fit{k}"
        fit_names.append(f"{pen}:{lam}")
        out[key + "_beta"] = r["beta"]
        out[key + "_objective"] = r["objective"]
        out[key + "_cycles"] = r["cycles"]
        out[key + "_converged"] = r["converged"]
        out[key + "_trace"] = r["objective_trace"]
        out[key + "_skipped"] = r["skipped_steps"]
        out[key + "_nonzero"] = r["nonzero_count"]
    out["fits"] = np.array(fit_names)
    if extra:
        out.update(extra)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(f"{name}: n={len(c['times'])} p={p} nnz={len(c['rows'])}")


def evaluate_strata(name, c, strata, model, beta_seed=11, beta_scale=0.3,
                    fits=(("l1", 0.5), ("none", 0.0)), max_cycles=200):
    """Composition oracle: sum of the reference over each stratum's rows."""
    p = c["n_cols"]
    rng = np.random.default_rng(beta_seed)
    beta = rng.uniform(-beta_scale, beta_scale, size=p)
    groups = [np.nonzero(strata == s)[0] for s in np.unique(strata)]
    parts = [ref_dataset(c, g) for g in groups]
    out = dict(c)
    out.update(model=model, beta_probe=beta, strata=strata)

    def derivs(b):
        g = np.zeros(p)
        h = np.zeros(p)
        for ds in parts:
            for j in range(p):
                gg, hh = ref.grad_hessian(ds, model, b, j, threads=1)
                g[j] += gg
                h[j] += hh
        return g, h

    def ll(b):
        return sum(ref.log_likelihood(ds, model, b, threads=1) for ds in parts)

    out["grad"], out["hess"] = derivs(beta)
    out["ll"] = ll(beta)
    out["ll0"] = ll(np.zeros(p))
    fit_names = []
    for k, (pen, lam) in enumerate(fits):
        kind = {"none": 0, "l1": 1, "l2": 2}[pen]
        b = np.zeros(p)
        hw = np.ones(p)

        def obj(b):
            pv = 0.0 if kind == 0 else (lam * np.abs(b).sum() if kind == 1
                                        else (b * b / (2 * lam)).sum())
            return ll(b) - pv
        prev = obj(b)
        trace = [prev]
        cycles = 0
        converged = False
        while not converged and cycles < max_cycles:
            cycles += 1
            for j in range(p):
                gj = sum(ref.grad_hessian(ds, model, b, j, threads=1)[0] for ds in parts)
                hj = sum(ref.grad_hessian(ds, model, b, j, threads=1)[1] for ds in parts)
                st = orc.coordinate_step(b[j], gj, hj, kind, lam, kind != 0, hw[j])
                if st["skipped"]:
                    continue
                b[j] = st["new_beta"]
                hw[j] = st["new_halfwidth"]
            o = obj(b)
            trace.append(o)
            converged = abs(o - prev) / max(1.0, abs(o)) < 1e-6
            prev = o
        key = f"fit{k}"
        fit_names.append(f"{pen}:{lam}")
        out[key + "_beta"] = b.copy()
        out[key + "_objective"] = prev
        out[key + "_cycles"] = cycles
        out[key + "_converged"] = converged
        out[key + "_trace"] = np.array(trace)
    out["fits"] = np.array(fit_names)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(f"{name}: n={len(c['times'])} p={p} strata={len(groups)}")


def known_answers():
    """Hand-checked cases from the reference unit tests."""
    cases = {}
    # test_engine.cpp:48-61 — times (2,1), both events, x=(1,0): g=-0.5 h=-0.25 fixed=1
    cases["two_subject"] = dict(times=np.array([2.0, 1.0]), status=np.array([1, 1]),
                                rows=np.array([0]), cols=np.array([0]),
                                values=np.array([1.0]), n_cols=1,
                                want_grad=-0.5, want_hess=-0.25, want_fixed=1.0)
    # test_engine.cpp:63-69 — uniform risk ll = -ln 6 (one covariate, all zero)
    cases["uniform_risk"] = dict(times=np.array([3.0, 2.0, 1.0]), status=np.array([1, 1, 1]),
                                 rows=np.zeros(0, np.int64), cols=np.zeros(0, np.int64),
                                 values=np.zeros(0), n_cols=1, want_ll=-np.log(6.0))
    # test_engine.cpp:71-83 — no events: exact zeros
    cases["no_events"] = dict(times=np.array([3.0, 2.0, 1.0]), status=np.array([0, 0, 0]),
                              rows=np.array([0]), cols=np.array([0]), values=np.array([1.0]),
                              n_cols=1, want_grad=0.0, want_hess=0.0, want_ll=0.0)
    # test_scan.cpp:271-289 shape as a dataset: times (3,3,1) all events,
    # x=(1,0,1), beta chosen so exp(eta)=(2,1,1) is not reachable with one
    # indicator; instead use the tied block with beta=0: D=(2,3), N1 = (1, 2)
    cases["tied_block"] = dict(times=np.array([3.0, 3.0, 1.0]), status=np.array([1, 1, 1]),
                               rows=np.array([0, 2]), cols=np.array([0, 0]),
                               values=np.array([1.0, 1.0]), n_cols=1,
                               # block {0,1}: D=2, G=1/2 (x2 events); row 2: D=3, G=2/3
                               want_grad=2.0 - (2 * 0.5 + 2.0 / 3.0),
                               want_hess=-(2 * (0.5 - 0.25) + (2.0 / 3.0 - 4.0 / 9.0)))
    for name, c in cases.items():
        ds = ref_dataset(c)
        p = c["n_cols"]
        g, h = ref.grad_hessian(ds, "cox", np.zeros(p), 0, threads=1)
        c["grad0"] = np.array([g])
        c["hess0"] = np.array([h])
        c["ll0"] = ref.log_likelihood(ds, "cox", np.zeros(p), threads=1)
        c["model"] = "cox"
        np.savez_compressed(os.path.join(HERE, f"ka_{name}.npz"), **c)
        print(f"ka_{name}: g={g} h={h} ll={c['ll0']}")


def main():
    known_answers()
    evaluate("cox_small", raw_case(250, 8, 0.15, 61), "cox")
    evaluate("cox_ties", raw_case(600, 10, 0.1, 62, quant=4.0, cens=0.4), "cox")
    evaluate("cox_valued", raw_case(400, 8, 0.12, 63, valued=True, dense_cols=2), "cox")
    evaluate("cox_nocens", raw_case(500, 12, 0.05, 64, cens=0.0), "cox")
    evaluate("fg_small", raw_case(220, 6, 0.2, 67, competing=0.3, cens=0.3), "finegray")
    evaluate("fg_ties", raw_case(500, 8, 0.15, 68, competing=0.25, quant=3.0, cens=0.4),
             "finegray")
    evaluate("fg_nocomp", raw_case(300, 5, 0.2, 69, cens=0.3), "finegray")
    # a reference-simulated design (simgen.cpp) extracted through the API
    sim, _ = ref.simulate_cox(n=400, p=6, density=0.2, seed=5, censoring_quantile=0.9)
    evaluate("cox_refsim", from_ref_sim(sim), "cox")
    fsim, _, _ = ref.simulate_finegray(n=400, p=6, density=0.2, seed=5,
                                       censoring_quantile=0.9)
    evaluate("fg_refsim", from_ref_sim(fsim), "finegray", fits=[("l1", 0.05), ("none", 0.0)])
    # multi-tile case for the GPU (TILE=4096 rows): several tiles, ties, censoring
    evaluate("cox_multitile", raw_case(20000, 40, 0.01, 71, quant=50.0, cens=0.3),
             "cox", fits=[("l1", 2 ** 0.5), ("l1", 40.0)])
    evaluate("fg_multitile", raw_case(12000, 20, 0.02, 72, competing=0.2, quant=50.0,
                                      cens=0.3), "finegray", fits=[("l1", 2 ** 0.5)])
    # strata (composition oracle)
    c = raw_case(900, 6, 0.15, 73, quant=5.0, cens=0.3)
    strata = np.random.default_rng(73).integers(0, 4, size=900)
    evaluate_strata("cox_strata", c, strata, "cox")
    c = raw_case(700, 5, 0.2, 74, competing=0.25, cens=0.3)
    strata = np.random.default_rng(74).integers(0, 3, size=700)
    evaluate_strata("fg_strata", c, strata, "finegray", fits=(("l1", 0.5),))


if __name__ == "__main__":
    main()
