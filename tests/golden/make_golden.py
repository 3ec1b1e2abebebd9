"""Generate the golden parity vectors from the UNMODIFIED reference package.

Run in the build container only (needs /root/reference, read-only):

    PYTHONPATH=/root/repo python tests/golden/make_golden.py

It imports ``momentcp`` from /root/reference/pkg/src, evaluates the reference on the seeded
instances of ``instances.py`` and writes the outputs (plus SHA-256 of the inputs) to
``tests/golden/*.npz``.  Nothing on the GPU box reads /root/reference; the tests compare the
oracle restatement and the CUDA path against these committed vectors.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)

import momentcp as ref  # noqa: E402  (the reference, read-only)
from momentcp.optimize import OptConfig, lbfgs_minimize, pack, packed_fg_implicit  # noqa: E402

import instances  # noqa: E402


def ref_obs(V, nu):
    return ref.ObservationSet(np.asarray(V, dtype=float), nu)


def term_scales(obs, lam, A, d, alpha):
    # exactly pkg/tests/test_acceptance.py:65-74, through the reference kernels
    oa = ref.ObservationSet(np.abs(obs.V), obs.nu)
    la, Aa = np.abs(lam), np.abs(A)
    Ya = ref.ttsv_batch(oa, Aa, d)
    cache = ref.build_gram_cache(la, Aa, d, Ya)
    f_s = abs(alpha) + float(la @ cache.u) + 2.0 * float(cache.w @ la)
    gl_s = 2.0 * (cache.w + cache.u)
    gA_s = 2.0 * d * (Ya + (Aa * la) @ cache.C) * la
    return f_s, gl_s, gA_s, Ya


def sweep(kind, count, make):
    out = {}
    for k in range(count):
        V, nu, lam, A, d, alpha = make(k)
        obs = ref_obs(V, nu)
        res = ref.fg_implicit(obs, lam, A, d, alpha)
        Y = ref.ttsv_batch(obs, A, d)
        w, _ = ref.model_data_inner(Y, A, lam)
        dn = ref.data_norm_sq(obs, d)
        f_s, gl_s, gA_s, Ya = term_scales(obs, lam, A, d, alpha)
        dn_s = ref.data_norm_sq(ref.ObservationSet(np.abs(obs.V), obs.nu), d)
        key = f"{kind}{k}_"
        out[key + "sha"] = np.array(instances.sha(V, lam, A) if nu is None
                                    else instances.sha(V, nu, lam, A, ))
        out[key + "f"] = np.array(res.f)
        out[key + "g_lam"] = res.g_lam
        out[key + "g_A"] = res.g_A
        out[key + "Y"] = Y
        out[key + "w"] = w
        out[key + "dnorm"] = np.array(dn)
        out[key + "f_scale"] = np.array(f_s)
        out[key + "gl_scale"] = gl_s
        out[key + "gA_scale"] = gA_s.astype(np.float32)   # scales only need 1e-7 accuracy
        out[key + "Y_scale"] = Ya.astype(np.float32)
        out[key + "dnorm_scale"] = np.array(dn_s)
        if V.shape[0] ** d <= 200_000:
            X = ref.build_moment(obs, d)
            re = ref.fg_explicit(X, lam, A, alpha)
            out[key + "f_explicit"] = np.array(re.f)
    return out


def kats():
    o = {}
    obs = ref.ObservationSet(np.array([[1.0], [2.0]]), np.array([1.0]))
    o["ttsv_9_18"] = ref.ttsv_batch(obs, np.array([[1.0], [1.0]]), 3)       # test_implicit.py:33-36
    o["dnorm_64"] = np.array(ref.data_norm_sq(
        ref.ObservationSet(np.array([[2.0]]), np.array([1.0])), 3))            # test_implicit.py:101-103
    w, val = ref.model_data_inner(np.array([[9.0], [18.0]]), np.array([[1.0], [1.0]]),
                                  np.array([1.0]))                            # test_implicit.py:128-133
    o["w_27"] = w
    v = np.array([0.6, 0.8])
    res = ref.fg_implicit(ref.ObservationSet(v[:, None], np.array([1.0])), np.array([1.0]),
                          v[:, None], 3, alpha=1.0)                           # test_objective.py:108-112
    o["exact_fit_f"] = np.array(res.f)
    model = ref.SymKruskal(3, np.array([2.0]), np.array([[1.0], [1.0]]))
    o["kruskal_32"] = np.array(ref.kruskal_norm_sq(model))                    # test_implicit.py:80-82
    return o


def configs():
    out = {}
    for name in instances.CONFIG_CASES:
        t0 = time.time()
        cfg, V, lam, A = instances.config_instance(name)
        obs = ref_obs(V, None)
        key = name + "_"
        out[key + "sha"] = np.array(instances.sha(V) if lam is None else instances.sha(V, lam, A))
        if cfg.r:
            res = ref.fg_implicit(obs, lam, A, cfg.d, 0.0)
            out[key + "f"] = np.array(res.f)
            out[key + "g_lam"] = res.g_lam
            out[key + "g_A"] = res.g_A
            if cfg.n * cfg.r <= 1000:
                out[key + "Y"] = ref.ttsv_batch(obs, A, cfg.d)
            f_s, gl_s, gA_s, Ya = term_scales(obs, lam, A, cfg.d, 0.0)
            out[key + "f_scale"] = np.array(f_s)
            out[key + "gl_scale"] = gl_s
            out[key + "gA_scale"] = gA_s.astype(np.float32)
        dn = ref.data_norm_sq(obs, cfg.d)
        out[key + "dnorm"] = np.array(dn)
        out[key + "dnorm_scale"] = np.array(
            ref.data_norm_sq(ref.ObservationSet(np.abs(obs.V), obs.nu), cfg.d))
        print(f"  {name}: p={V.shape[1]} {time.time() - t0:.1f}s", flush=True)
    return out


def lbfgs_c1():
    """100-iteration reference L-BFGS fit at c1 (BASELINE configs[0]), every iterate kept."""
    cfg, V, lam, A = instances.config_instance("c1")
    obs = ref_obs(V, None)
    fg = packed_fg_implicit(obs, cfg.d, cfg.r)
    iterates = []
    rep = lbfgs_minimize(fg, pack(lam, A), OptConfig(max_iters=100), shape=(cfg.n, cfg.r),
                         iterate_hook=iterates.append)
    X = np.stack(iterates)
    fvals = np.array([fg(x)[0] for x in X])
    return {"iterates": X, "f": fvals, "final_f": np.array(rep.f), "n_fg": np.array(rep.n_fg),
            "n_steps": np.array(rep.n_steps), "reason": np.array(rep.reason),
            "final_lam": rep.lam, "final_A": rep.A, "grad_inf": np.array(rep.grad_inf_norm)}


def adam_c1():
    """Reference epoch-based Adam at c1 (small epochs so the run ends by itself)."""
    from momentcp.optimize import AdamConfig, adam_minimize

    cfg, V, lam, A = instances.config_instance("c1")
    obs = ref_obs(V, None)
    rep = adam_minimize(obs, cfg.d, cfg.r, pack(lam, A), AdamConfig(**instances.ADAM_C1),
                        np.random.default_rng(instances.ADAM_SEED))
    return {"trace_f": np.array([t[0] for t in rep.trace]), "final_f": np.array(rep.f),
            "n_fg": np.array(rep.n_fg), "reason": np.array(rep.reason), "final_lam": rep.lam,
            "final_A": rep.A, "grad_inf": np.array(rep.grad_inf_norm)}


def main():
    if sys.argv[1:] == ["adam"]:
        np.savez_compressed(os.path.join(HERE, "adam_c1.npz"), **adam_c1())
        return
    t = time.time()
    np.savez_compressed(os.path.join(HERE, "kat.npz"), **kats())
    sw = sweep("t", instances.TINY_COUNT, instances.tiny_instance)
    sw.update(sweep("e", instances.EXT_COUNT, instances.ext_instance))
    np.savez_compressed(os.path.join(HERE, "sweep.npz"), **sw)
    print(f"sweep done {time.time() - t:.1f}s", flush=True)
    np.savez_compressed(os.path.join(HERE, "configs.npz"), **configs())
    np.savez_compressed(os.path.join(HERE, "lbfgs_c1.npz"), **lbfgs_c1())
    np.savez_compressed(os.path.join(HERE, "adam_c1.npz"), **adam_c1())
    print(f"all done {time.time() - t:.1f}s")


if __name__ == "__main__":
    main()
