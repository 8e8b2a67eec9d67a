"""Generate golden vectors from the reference package (build container only).

Run from the repo root:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the *unmodified* reference ``dtopk`` package read-only from
/root/reference/pkg/src, runs it on seeded inputs made by the reference's own
generators (data.gen_uniform / gen_normal / gen_customized, data.py:58-113)
and writes inputs + outputs to ``tests/golden/golden.npz``.  The fixtures
travel with the repo; /root/reference does not exist on the GPU box.

Recorded per case: input keys, k, the config as resolved by
validate_config (core.py:145-174), ``dr_topk`` values / threshold / all
WorkloadStats counters (pipeline.py:172-220), the delegate vector
(delegate.py:142-155) and the first_topk threshold for both skip_last
settings (pipeline.py:87-116).  float32 and smallest cases go through the
order-preserving key map the reference README names as its extension point
(pkg/README.md:108-110); their expected outputs are mapped back.
"""

from __future__ import annotations

import json
import pathlib
import sys
from dataclasses import replace

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import dtopk  # noqa: E402
from dtopk import data  # noqa: E402
from dtopk.pipeline import first_topk  # noqa: E402

OUT = pathlib.Path(__file__).with_name("golden.npz")


def f32_keys(v: np.ndarray, largest: bool) -> np.ndarray:
    b = v.view(np.uint32)
    u = np.where(b >> np.uint32(31), ~b, b | np.uint32(0x80000000)).astype(np.uint32)
    return u if largest else ~u


def f32_from_keys(u: np.ndarray, largest: bool) -> np.ndarray:
    u = u if largest else ~u
    b = np.where(u & np.uint32(0x80000000), u ^ np.uint32(0x80000000), ~u).astype(np.uint32)
    return b.view(np.float32)


def cases():
    rng = np.random.default_rng(20261017)
    # (name, input, k, cfg kwargs)
    for seed in range(3):
        yield f"ud16_s{seed}", data.gen_uniform(2**16, seed), 128, {}
        yield f"nd14_s{seed}", data.gen_normal(2**14, seed), 200, {}
        yield f"cd14_s{seed}", data.gen_customized(2**14, 2**10, seed), 2**10, {}
    yield "ud16_k1", data.gen_uniform(2**16, 7), 1, {}
    yield "ud16_k4096", data.gen_uniform(2**16, 8), 4096, {}
    yield "ud_odd", data.gen_uniform(50_001, 9), 333, {}
    yield "ud_beta1", data.gen_uniform(2**15, 10), 256, {"beta": 1}
    yield "ud_beta3", data.gen_uniform(2**15, 11), 256, {"beta": 3}
    yield "ud_alpha3", data.gen_uniform(2**14, 12), 100, {"alpha": 3, "auto_alpha": False}
    yield "ud_alpha14", data.gen_uniform(2**16, 13), 2, {"alpha": 14, "auto_alpha": False}
    yield "fewdistinct", rng.integers(0, 16, 2**15, dtype=np.uint32), 2**10, {}
    yield "allequal", np.full(2**14, 0x5A5A5A5A, dtype=np.uint32), 777, {}
    yield "ascending", np.arange(2**15, dtype=np.uint32), 2**9, {}
    yield "descending", np.arange(2**15, dtype=np.uint32)[::-1].copy(), 2**9, {}
    yield "fallback", data.gen_uniform(1024, 14), 600, {"alpha": 8, "beta": 2, "auto_alpha": False}
    yield "k_eq_n", data.gen_uniform(1024, 15), 1024, {}
    yield "small_tail", rng.integers(0, 50, 77, dtype=np.uint32), 5, {"alpha": 4, "auto_alpha": False}


def fcases():
    g = np.random.Generator(np.random.Philox(99))
    yield "f32_normal", g.standard_normal(2**15, dtype=np.float32), 2**8
    yield "f32_pareto", g.pareto(1.5, 2**15).astype(np.float32), 2**8
    z = g.standard_normal(2**12, dtype=np.float32)
    z[::7] = 0.0
    z[::11] = -0.0
    yield "f32_zeros", z, 100


def main():
    arrays = {}
    meta = []
    for name, v, k, kw in cases():
        v = np.ascontiguousarray(v, dtype=np.uint32)
        cfg = dtopk.validate_config(dtopk.PipelineConfig(k=k, **kw), v.size)
        entry = {"name": name, "kind": "u32", "k": k, "cfg": kw, "alpha": cfg.alpha, "beta": cfg.beta,
                 "direct": bool(cfg.direct_fallback)}
        arrays[f"{name}__input"] = v
        for sl in (True, False):
            st = dtopk.WorkloadStats()
            r = dtopk.dr_topk(v, replace(dtopk.PipelineConfig(k=k, **kw), skip_last_iteration=sl), stats=st)
            tag = "sl1" if sl else "sl0"
            arrays[f"{name}__values_{tag}"] = r.values
            entry[f"threshold_{tag}"] = int(r.threshold)
            entry[f"stats_{tag}"] = {
                "delegate_vector_len": st.delegate_vector_len,
                "concatenated_len": st.concatenated_len,
                "fully_qualified_subranges": st.fully_qualified_subranges,
                "partially_qualified_subranges": st.partially_qualified_subranges,
                "elements_read": st.elements_read,
                "elements_written": st.elements_written,
            }
        if not cfg.direct_fallback:
            d = dtopk.extract_delegates(v, cfg.alpha, cfg.beta)
            arrays[f"{name}__delegates"] = d.values
            for sl in (True, False):
                rep = first_topk(d, k, "radix", skip_last=sl)
                entry[f"theta_{'sl1' if sl else 'sl0'}"] = int(rep.theta)
        meta.append(entry)
    for name, v, k in fcases():
        for largest in (True, False):
            keys = f32_keys(v, largest)
            r = dtopk.dr_topk(keys, dtopk.PipelineConfig(k=k))
            tag = f"{name}_{'max' if largest else 'min'}"
            arrays[f"{tag}__input"] = v
            arrays[f"{tag}__values_sl1"] = f32_from_keys(r.values, largest)
            meta.append({"name": tag, "kind": "f32", "largest": largest, "k": k, "cfg": {},
                         "threshold_sl1": float(f32_from_keys(np.array([r.threshold], np.uint32), largest)[0])})
    arrays["__meta__"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(meta)} cases)")


if __name__ == "__main__":
    main()
