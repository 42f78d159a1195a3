"""Generate tests/golden/gating_golden.json from the REFERENCE itself.

Runs the reference's routing code compiled verbatim (oracle/_ref/
libmoesim_ref.so, built by `make -C oracle` from /root/reference/proj/src) on:

* every hand-written golden case of proj/tests/test_gating.cpp (with the
  expected values the reference test asserts, copied as data), and
* the randomized suites of test_gating.cpp / acceptance.cpp, replayed
  bit-exactly with std::mt19937_64 (tests/refrng.py) -- for those the fixture
  stores a SHA-256 digest of the reference's outputs per suite, plus the full
  outputs of the first few cases.

Usage (in the dev container, where /root/reference exists):
    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import native as N  # noqa: E402
from refrng import MT19937_64, experts_array, random_batch  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "gating_golden.json")


def digest(arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.int64).tobytes())
        h.update(b"|")
    return h.hexdigest()


def dyn(ex, E):
    o, c, s = N.ref_dynamic_dispatch(ex, E)
    return {"order": o.tolist(), "counts": c.tolist(), "splits": s.tolist()}


def sta(ex, E, C):
    cap, slots, dropped = N.ref_static_dispatch(ex, E, C)
    return {"capacity": cap, "slots": slots.tolist(), "dropped": dropped.tolist()}


def explicit_cases():
    k1 = lambda ids: np.array(ids, np.int32).reshape(-1, 1)  # noqa: E731
    cases = []
    # test_gating.cpp:64-77
    cases.append({"src": "test_gating.cpp:64-77", "kind": "static", "experts": [[2], [0], [1], [0], [2], [0]],
                  "E": 3, "C": 0.5, "expect": sta(k1([2, 0, 1, 0, 2, 0]), 3, 0.5)})
    # :79-85
    cases.append({"src": "test_gating.cpp:79-85", "kind": "static", "experts": [[0], [0], [0], [0], [1], [2]],
                  "E": 3, "C": 0.5, "expect": sta(k1([0, 0, 0, 0, 1, 2]), 3, 0.5)})
    # :87-95
    cases.append({"src": "test_gating.cpp:87-95", "kind": "static", "experts": [[0], [1]], "E": 2, "C": 1.0,
                  "expect": sta(k1([0, 1]), 2, 1.0)})
    # :132-138
    cases.append({"src": "test_gating.cpp:132-138", "kind": "dynamic", "experts": [[2], [0], [1], [0], [2], [0]],
                  "E": 3, "expect": dyn(k1([2, 0, 1, 0, 2, 0]), 3)})
    # :140-147
    cases.append({"src": "test_gating.cpp:140-147", "kind": "dynamic", "experts": [[0], [0], [0], [0]], "E": 4,
                  "expect": dyn(k1([0, 0, 0, 0]), 4)})
    # :149-158
    cases.append({"src": "test_gating.cpp:149-158", "kind": "dynamic", "experts": [[0, 1], [1, 0]], "E": 2,
                  "expect": dyn(np.array([[0, 1], [1, 0]], np.int32), 2)})
    # :292-302 debug_json golden strings
    cases.append({"src": "test_gating.cpp:292-302", "kind": "debug_json_dynamic", "experts": [[1], [0], [1]],
                  "E": 2, "expect": N.ref_debug_json(k1([1, 0, 1]), 2)})
    cases.append({"src": "test_gating.cpp:292-302", "kind": "debug_json_static", "experts": [[1], [0], [1]],
                  "E": 2, "C": 1.0 / 3.0, "expect": N.ref_debug_json(k1([1, 0, 1]), 2, 1.0 / 3.0, True)})
    return cases


def scalar_goldens():
    lib = N.ref_lib()
    caps = [(0.5, 6), (0.05, 2048), (0.1, 30), (1.0, 128), (0.3, 5), (0.05, 16384), (1.0, 6144),
            (1.0 / 3.0, 3), (0.25, 7), (2.5, 3)]
    return {
        "expert_capacity": [[c, s, lib.ref_expert_capacity(c, s)] for c, s in caps],
        "waste_factor": [[e, c, k, lib.ref_waste_factor(e, c, k)] for e, c, k in
                         [(512, 0.05, 2), (128, 1.0, 2), (16, 2.0 / 16.0, 2)]],
        "dispatch_mask_elements": [[s, e, c, int(lib.ref_dispatch_mask_elements(s, e, c))] for s, e, c in
                                   [(6, 3, 0.5), (1, 1, 1.0), (2048, 512, 0.05), (16384, 512, 0.05)]],
    }


def random_suites():
    suites = []

    def suite(name, src, seed, iters, gen, keep=3):
        rng = MT19937_64(seed)
        arrays, first = [], []
        n = 0
        for _ in range(iters):
            item = gen(rng)
            if item is None:
                continue
            kind, ex, E, C = item
            if kind == "dynamic":
                o, c, s = N.ref_dynamic_dispatch(ex, E)
                arrays += [o, c, s]
                rec = {"E": E, "experts": ex.tolist(), "order": o.tolist(), "counts": c.tolist(),
                       "splits": s.tolist()}
            else:
                cap, slots, dropped = N.ref_static_dispatch(ex, E, C)
                arrays += [np.array([cap]), slots.reshape(-1), dropped.reshape(-1)]
                rec = {"E": E, "C": C, "experts": ex.tolist(), "capacity": cap, "slots": slots.tolist(),
                       "dropped": dropped.tolist()}
            if len(first) < keep:
                first.append(rec)
            n += 1
        suites.append({"name": name, "src": src, "seed": seed, "iters": iters, "cases": n,
                       "digest": digest(arrays), "first": first})

    # test_gating.cpp:105-130 drop law, seed 2024 (iteration consumes rng as the test does)
    def g_drop(rng):
        E = 2 + rng() % 8
        k = 1 + rng() % 2
        S = 1 + rng() % 40
        C = 0.05 + (rng() % 100) / 100.0
        if k > E:
            return None
        b = random_batch(rng, S, E, k)
        return ("static", experts_array(b), E, C)

    suite("drop_law", "test_gating.cpp:105-130", 2024, 500, g_drop)

    # test_gating.cpp:160-182 dynamic vs scan_group, seed 7
    def g_dyn(rng):
        E = 2 + rng() % 16
        k = 1 + rng() % 2
        S = 1 + rng() % 60
        b = random_batch(rng, S, E, k)
        return ("dynamic", experts_array(b), E, 0.0)

    suite("dynamic_scan", "test_gating.cpp:160-182", 7, 300, g_dyn)

    # acceptance.cpp:140-164 routing equivalence, seed 1001, S<=256, E<=32
    def g_acc(rng):
        E = 2 + rng() % 31
        k = 1 + rng() % 2
        S = 1 + rng() % 256
        b = random_batch(rng, S, E, k)
        return ("dynamic", experts_array(b), E, 0.0)

    suite("acceptance_routing", "acceptance.cpp:140-164 (shape ranges)", 1001, 1000, g_acc)
    return suites


def main():
    golden = {
        "generator": "tests/golden/make_golden.py",
        "reference": "oracle/_ref/libmoesim_ref.so built verbatim from /root/reference/proj/src",
        "explicit": explicit_cases(),
        "scalars": scalar_goldens(),
        "random": random_suites(),
    }
    with open(OUT, "w") as f:
        json.dump(golden, f, separators=(",", ":"))
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes)")


if __name__ == "__main__":
    main()
