"""Writes spec_examples.json: the known-answer examples the reference ships for
this path (SPEC.md; the reference has no test files).  Each entry
cites its SPEC.md line.  Values are transcribed from the spec text; the dense
PageRank oracle value for the 3-chain is computed here with numpy (the spec
says "compare against a dense-matrix power-iteration oracle").

Run:  python tests/golden/make_spec_examples.py
"""
import json
import os

import numpy as np

NO_REF = None


def dense_pagerank(n, edges, alpha, iters, dangling="uniform"):
    A = np.zeros((n, n))
    for u, v in edges:
        A[u, v] = 1.0
    d = A.sum(axis=1)
    p0 = np.full(n, 1.0 / n)
    p = p0.copy()
    for _ in range(iters):
        q = np.where(d > 0, p / np.where(d > 0, d, 1), 0.0)
        D = p[d == 0].sum()
        y = A.T @ q
        p = alpha * p0 + (1 - alpha) * (y + (D / n if dangling == "uniform" else 0.0))
    return p.tolist()


ex = {
    "build_csr": [
        {"spec": "SPEC.md:52", "n": 3, "edges": [], "rows": [[], [], []]},
        {"spec": "SPEC.md:53", "n": 2, "edges": [[0, 1], [0, 1], [1, 0]], "rows": [[1], [0]]},
        {"spec": "SPEC.md:54", "n": 3, "edges": [[0, 2], [0, 1], [1, 2]], "rows": [[1, 2], [2], []]},
    ],
    "transpose": [
        {"spec": "SPEC.md:62", "rows": [], "want": []},
        {"spec": "SPEC.md:63", "rows": [[1], []], "want": [[], [0]]},
    ],
    "out_degrees": [
        {"spec": "SPEC.md:72", "rows": [[], [], [], []], "want": [0, 0, 0, 0]},
        {"spec": "SPEC.md:73", "rows": [[1, 2], [0, 2], [0, 1]], "want": [2, 2, 2]},
    ],
    "matvec_csr": [
        {"spec": "SPEC.md:84", "rows": [[1, 2], [2], []], "x": [1, 2, 3], "y": [5, 3, 0]},
        {"spec": "SPEC.md:83", "rows": [[0], [1], [2], [3]], "x": [0.5, 0.25, 2.0, -1.0], "y": [0.5, 0.25, 2.0, -1.0]},
        {"spec": "SPEC.md:82", "rows": [[1, 2], [0], [0, 1, 2]], "x": [0, 0, 0], "y": [0, 0, 0]},
    ],
    "compress": [
        {"spec": "SPEC.md:135", "rows": [[1, 2], [1, 2, 3], [], []], "window": 1,
         "refs": [NO_REF, 0, NO_REF, NO_REF], "plus": [[1, 2], [3], [], []], "minus": [[], [], [], []],
         "m_prime": 3},
        {"spec": "SPEC.md:136", "rows": [[], [], []], "window": 2, "refs": [NO_REF] * 3, "plus": [[], [], []],
         "minus": [[], [], []], "m_prime": 0},
        {"spec": "SPEC.md:137", "rows": [[5], [9]] + [[]] * 8, "window": 1, "refs": [NO_REF] * 10,
         "plus": [[5], [9]] + [[]] * 8, "minus": [[]] * 10, "m_prime": 2},
    ],
    "reconstruct_row": [
        {"spec": "SPEC.md:146", "n": 4, "refs": [NO_REF, 0, NO_REF, NO_REF], "plus": [[1, 2], [3], [], []],
         "minus": [[], [], [], []], "row": 1, "want": [1, 2, 3]},
    ],
    "stats": [
        {"spec": "SPEC.md:155", "rows": [[], []], "window": 1, "m": 0, "m_prime": 0, "ratio": 1.0,
         "ratio_by_convention": True},
        {"spec": "SPEC.md:156", "rows": [[1, 2], [1, 2, 3], [], []], "window": 1, "m": 5, "m_prime": 3,
         "ratio": 5 / 3, "ratio_by_convention": False},
    ],
    "matvec_ref": [
        {"spec": "SPEC.md:204", "n": 4, "refs": [NO_REF, 0, NO_REF, NO_REF], "plus": [[1, 2], [3], [], []],
         "minus": [[], [], [], []], "x": [1, 1, 1, 1], "y": [2, 3, 0, 0], "adds": 4},
        {"spec": "SPEC.md:205", "n": 2, "refs": [NO_REF, 0], "plus": [[0, 1], []], "minus": [[], [0]],
         "x": [2, 5], "y": [7, 5], "adds": 4},
    ],
    "matvec_ref_left": [
        {"spec": "SPEC.md:214", "rows": [[1], []], "x": [1, 0], "y": [0, 1]},
        {"spec": "SPEC.md:213", "rows": [[0], [1], [2]], "x": [3, 4, 5], "y": [3, 4, 5]},
    ],
    "pagerank": [
        {"spec": "SPEC.md:261", "n": 2, "edges": [[0, 1], [1, 0]], "alpha": 0.15, "iterations": 10,
         "dangling": "uniform", "want": [0.5, 0.5], "tol": 1e-12},
        {"spec": "SPEC.md:263", "n": 3, "edges": [[0, 1], [1, 2]], "alpha": 0.15, "iterations": 50,
         "dangling": "uniform", "want": dense_pagerank(3, [[0, 1], [1, 2]], 0.15, 50), "tol": 1e-10},
    ],
    # biclique module (reference include/cmv/biclique.hpp)
    "matvec_biclique": [
        {"spec": "SPEC.md:317", "n": 4, "bicliques": [[[0, 1], [2, 3]]], "residual": [], "x": [0, 0, 1, 1],
         "c": [2], "y": [2, 2, 0, 0], "adds": 4, "m": 4},
        {"spec": "SPEC.md:318", "n": 6, "bicliques": [[[0, 1, 2], [3, 4, 5]]], "residual": [],
         "x": [0, 0, 0, 1, 1, 1], "c": [3], "y": [3, 3, 3, 0, 0, 0], "adds": 6, "m": 9},
        {"spec": "SPEC.md:316", "n": 3, "bicliques": [], "residual": [[0, 1], [1, 2], [2, 0]], "x": [1, 2, 3],
         "c": [], "y": [2, 3, 1], "adds": 3, "m": 3},
    ],
    "extract_greedy": [
        {"spec": "SPEC.md:326", "n": 6, "edges": [[u, v] for u in range(3) for v in range(3, 6)],
         "bicliques": [[[0, 1, 2], [3, 4, 5]]], "residual": [], "compressed_size": 6, "m": 9},
        {"spec": "SPEC.md:328", "n": 8, "edges": sorted({(u, v) for u in range(3) for v in range(4, 8)}
                                                        | {(u, v) for u in range(1, 4) for v in range(5, 8)}),
         "verify": True},
    ],
    "verify_cover": [
        {"spec": "SPEC.md:335", "n": 3, "edges": [[0, 1], [1, 2]], "bicliques": [], "residual": [[0, 1], [1, 2]],
         "want": True},
        {"spec": "SPEC.md:337", "n": 4, "edges": [[0, 2], [0, 3], [1, 2], [1, 3]], "bicliques": [[[0, 1], [2, 3]]],
         "residual": [[0, 2]], "want": False},
    ],
}

if __name__ == "__main__":
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "spec_examples.json")
    with open(out, "w") as f:
        json.dump(ex, f, indent=1)
    print("wrote", out)
