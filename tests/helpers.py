"""Shared test helpers: golden-vector loaders, tolerance checks, batch builders."""

from __future__ import annotations

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"

# relative tolerances stated by the north star (BASELINE.json): <= 1e-5 in
# fp32 mode, <= 2e-2 in bf16; f64 mode (the reference's own precision) is
# held to 1e-12.  Checked normwise per array (max-abs error over max-abs
# reference) AND on the delta alone, where the output's own rounding (one
# ulp of the stored element) is allowed on top.
REL_TOL = {"f64": 1e-12, "f32": 1e-5, "bf16": 2e-2}
OUT_ULP = {"f64": 2.0**-52, "f32": 2.0**-23, "bf16": 2.0**-8}


def load(name: str):
    return np.load(GOLDEN / name, allow_pickle=False)


def mask_batches():
    g = load("masks.npz")
    e_off, t_off = g["e_off"], g["t_off"]
    out = []
    qpos = 0
    for i in range(len(e_off) - 1):
        e0, e1 = e_off[i], e_off[i + 1]
        E = e1 - e0
        qsl = g["qsl"][qpos : qpos + E + 1]
        qpos += E + 1
        out.append(
            dict(
                qsl=qsl,
                adapter=g["adapter"][e0:e1],
                is_decode=g["is_decode"][e0:e1],
                all_pos=g["all_pos"][e0:e1],
                prompt_len=g["prompt_len"][e0:e1],
                cache_start=g["cache_start"][e0:e1],
                mask=g["mask"][t_off[i] : t_off[i + 1]],
                uniform={1: True, 0: False, -1: None}[int(g["uniform"][i])],
            )
        )
    return out


def delta_cases():
    g = load("deltas.npz")
    out = []
    for i in range(int(g["n_cases"])):
        k = f"c{i:03d}_"
        c = {name[len(k):]: g[name] for name in g.files if name.startswith(k)}
        c["kind"] = str(c["kind"])
        c["rank"] = int(c["rank"])
        c["s"] = float(c["s"])
        c["dims"] = tuple(int(v) for v in c["dims"])
        out.append(c)
    return out


def masked_cases():
    g = load("masked.npz")
    out = []
    for i in range(int(g["n_cases"])):
        k = f"m{i:03d}_"
        c = {name[len(k):]: g[name] for name in g.files if name.startswith(k)}
        c["kind"] = str(c["kind"])
        c["s"] = float(c["s"])
        c["rank"] = int(c["rank"])
        c["plen"] = int(c["plen"])
        c["sched_all"] = bool(c["sched_all"])
        c["dims"] = tuple(int(v) for v in c["dims"])
        out.append(c)
    return out


def params_of(c: dict) -> dict:
    return {k: c[k] for k in ("A", "B", "b", "R", "W") if k in c}


def make_params(c: dict):
    """A package AdapterParams from a golden case dict (scaling = constant s
    reproduces the reference prefactor exactly)."""
    from paper_2605_14217_b200 import AdapterKind, AdapterParams, ScalingRule

    kind = AdapterKind(c["kind"])
    return AdapterParams(kind, c["rank"], c["dims"], ScalingRule.constant(c["s"]), **params_of(c))


def check_close(out, base, ref, mode: str, what: str = ""):
    """Normwise + delta-wise tolerance check of an updated array."""
    out = np.asarray(out, dtype=np.float64)
    base = np.asarray(base, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    tol = REL_TOL[mode]
    scale = max(np.max(np.abs(ref)), 1e-300)
    err = np.max(np.abs(out - ref)) if out.size else 0.0
    assert err <= tol * scale, f"{what}: max|out-ref| {err:.3e} > {tol:g} * {scale:.3e}"
    d_out = out - base
    d_ref = ref - base
    dscale = np.max(np.abs(d_ref)) if d_ref.size else 0.0
    bound = tol * dscale + OUT_ULP[mode] * np.abs(ref) + 1e-300
    bad = np.abs(d_out - d_ref) > bound
    assert not bad.any(), (
        f"{what}: delta mismatch at {int(bad.sum())} elements, worst "
        f"{np.max(np.abs(d_out - d_ref)):.3e} vs delta scale {dscale:.3e}"
    )


# ---------------------------------------------------------------- BASELINE config 1 at its stated size

CFG1_D = 4096


def config1_full(shuffle: bool):
    """BASELINE configs[0] exactly, regenerated with this package's restated
    seeded constructors (bit-identical to the reference's, pinned by
    test_host_api / test_reference_live) in the order make_golden.py
    gen_config1_full uses: entries, adapters (init_zero_delta + perturbation,
    sigma 0.1), then x, h from rng_from_seed(0, 1).  Returns the golden file's
    arrays too (sampled reference rows + sha256 of the full outputs)."""
    from paper_2605_14217_b200.adapters import AdapterKind, init_zero_delta
    from paper_2605_14217_b200.batch import _perturbed_params
    from paper_2605_14217_b200.linalg import rng_from_seed

    g = load(f"config1_full{'_shuffled' if shuffle else ''}.npz")
    d = CFG1_D
    params = {}
    for a in range(32):
        kind, r, dims = (AdapterKind.DIREFT, 8, (d,)) if a < 16 else (AdapterKind.LORA, 1, (d, d))
        params[a] = _perturbed_params(init_zero_delta(kind, r, dims, a), a + 1000, 0.1)
    T = int(g["qsl"][-1])
    rng = rng_from_seed(0, 1)
    x = rng.normal(size=(T, d))
    h = rng.normal(size=(T, d))
    return g, params, x, h


def oracle_params(p) -> dict:
    """Oracle kwargs of an AdapterParams bundle (its own float64 operands)."""
    kw = {k: getattr(p, k) for k in ("A", "B", "b", "R", "W") if getattr(p, k) is not None}
    return dict(kind=p.kind.value, s=float(p.prefactor), **kw)
