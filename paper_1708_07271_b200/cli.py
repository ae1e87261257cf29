"""Command-line surface of the reference's cli-io module:
edge-list ingestion (`load_edge_list`) and the subcommands
`gen`, `compress`, `stats`, `matvec`, `pagerank`, `bench` and
`biclique-extract`, with the Table-1 style TSV report of
`run_bench`.  Exit code 0 on success, nonzero with a message
on any error.

    python -m paper_1708_07271_b200 gen --model copy --n 100000 --degree 12 --out g.txt
    python -m paper_1708_07271_b200 compress --window 7 --out g.cbv g.txt
    python -m paper_1708_07271_b200 stats g.cbv
    python -m paper_1708_07271_b200 matvec --uniform --seed 1 g.cbv
    python -m paper_1708_07271_b200 pagerank --alpha 0.15 --iters 50 --kernel ref g.txt
    python -m paper_1708_07271_b200 bench --reps 3 g.txt h.txt

Graphs are given as an edge-list text file (two 0-based ids per line, `#`
comments) or, for the commands that accept it, a CBV1 container (`.cbv`).
The products and PageRank run on the GPU through the library's kernels; there
is no CPU product path."""
from __future__ import annotations

import argparse
import os
import sys
import time
from typing import List, Optional

import numpy as np

from . import (UNBOUNDED_ROUNDS, BicliqueCover, BicliqueKernel, BvGpuKernel, BvGraph, BvParams, BvStream, CreateOptions, CsrGraph,
               DanglingPolicy, PageRankConfig, compression_stats, csr_matvec_device, pagerank,
               pagerank_equivalence_check)


class EdgeListError(ValueError):
    """Malformed edge-list line (parse error with line number)."""


def build_csr(edges: np.ndarray, n: int) -> CsrGraph:
    """cmv::build_csr (csr.hpp:39-41): rows sorted, duplicate
    edges collapsed, self-loops kept."""
    edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    if len(edges) and (edges.min() < 0 or edges.max() >= n):
        raise IndexError("build_csr: vertex id out of range")
    key = np.unique(edges[:, 0] * max(n, 1) + edges[:, 1]) if len(edges) else np.zeros(0, np.int64)
    src, dst = key // max(n, 1), key % max(n, 1)
    ro = np.zeros(n + 1, dtype=np.uint64)
    np.add.at(ro, src + 1, 1)
    ro = np.cumsum(ro, dtype=np.uint64)
    return CsrGraph.from_arrays(n, ro, dst.astype(np.uint32))


def load_edge_list(path: str, n: Optional[int] = None) -> CsrGraph:
    """load_edge_list: `#` comments and blank lines skipped;
    each data line holds two nonnegative integers; n = max id + 1 unless given;
    a malformed line raises EdgeListError naming its line number, an id >= n an
    IndexError."""
    src = sys.stdin if path == "-" else open(path, "r")
    rows: List[int] = []
    try:
        for ln, line in enumerate(src, 1):
            s = line.split("#", 1)[0].strip()
            if not s:
                continue
            parts = s.split()
            if len(parts) != 2 or not (parts[0].isdigit() and parts[1].isdigit()):
                raise EdgeListError(f"line {ln}: expected two nonnegative integers, got {line.rstrip()!r}")
            rows.append(int(parts[0]))
            rows.append(int(parts[1]))
    finally:
        if src is not sys.stdin:
            src.close()
    e = np.array(rows, dtype=np.int64).reshape(-1, 2)
    top = int(e.max()) + 1 if len(e) else 0
    if n is None:
        n = top
    elif top > n:
        raise IndexError(f"edge list: vertex id {top - 1} >= declared n = {n}")
    return build_csr(e, n)


def save_edge_list(g: CsrGraph, path: str) -> None:
    ro, co = g.row_offsets, g.columns
    src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(ro.astype(np.int64)))
    with open(path, "w") as f:
        f.write(f"# n={g.n} m={g.m}\n")
        np.savetxt(f, np.stack([src, co.astype(np.int64)], axis=1), fmt="%d")


def erdos_renyi(n: int, mean_degree: float, seed: int) -> CsrGraph:
    """Seeded Erdos-Renyi graph G(n, p = mean_degree / n) (`gen`)."""
    rng = np.random.default_rng(seed)
    m = rng.binomial(n * n, min(1.0, mean_degree / max(n, 1))) if n else 0
    e = rng.integers(0, max(n, 1), size=(m, 2), dtype=np.int64)
    return build_csr(e, n)


def _graph(path: str, n: Optional[int] = None) -> CsrGraph:
    if path.endswith(".cbv"):
        return BvStream.load(path).decode_host()
    return load_edge_list(path, n)


def _stream(path: str, window: int) -> BvStream:
    if path.endswith(".cbv"):
        return BvStream.load(path)
    return BvStream.encode(load_edge_list(path), BvParams(window=window))


def _vector(args, n: int) -> np.ndarray:
    if args.vector:
        x = np.loadtxt(args.vector, dtype=np.float64, ndmin=1)
        if x.shape != (n,):
            raise ValueError(f"vector has {x.size} entries, the graph has n = {n}")
        return x
    rng = np.random.default_rng(args.seed)
    return (rng.integers(0, 2 ** 64, size=n, dtype=np.uint64) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def cmd_gen(a) -> None:
    if a.model == "copy":
        g = CsrGraph.copy_model(a.n, a.degree, a.p_ref, a.p_copy, seed=a.seed)
    elif a.model == "social":
        g = CsrGraph.social(a.n, seed=a.seed)
    else:
        g = erdos_renyi(a.n, a.degree, a.seed)
    if a.out.endswith(".cbv"):
        BvStream.encode(g, BvParams(window=a.window)).save(a.out)
    else:
        save_edge_list(g, a.out)
    print(f"gen\t{a.model}\tn={g.n}\tm={g.m}\t{a.out}")


def cmd_compress(a) -> None:
    g = load_edge_list(a.graph, a.n)
    s = BvStream.encode(g, BvParams(window=a.window, max_ref=a.max_ref))
    s.save(a.out)
    st = s.stats()
    print(f"compress\tn={g.n}\tm={g.m}\tbits={st['stream_bits']}\tbits_per_edge={st['stream_bits'] / max(g.m, 1):.3f}"
          f"\t{a.out}")


def cmd_stats(a) -> None:
    s = _stream(a.graph, a.window)
    c = compression_stats(s)
    print("n\tm\tm_prime\tratio\tratio_by_convention\trows_self_coded\tmax_chain\tstream_bits")
    print(f"{c.n}\t{c.m}\t{c.m_prime}\t{c.ratio:.4f}\t{int(c.ratio_by_convention)}\t{c.rows_self_coded}\t{c.max_chain}"
          f"\t{s.stats()['stream_bits']}")


def cmd_matvec(a) -> None:
    s = _stream(a.graph, a.window)
    x = _vector(a, s.n)
    dg = BvGraph(s, CreateOptions(device=a.device))
    y = dg.matvec(x, form=a.form)
    if a.out:
        np.savetxt(a.out, y, fmt="%.17g")
    print(f"matvec\tform={a.form}\tn={s.n}\tm={s.m}\tsum={float(np.sum(y)):.17g}\tmax={float(np.max(y)) if s.n else 0:.17g}")


def _power_iteration(multiply, deg: np.ndarray, cfg: PageRankConfig):
    """The reference's pagerank recurrence (pagerank.hpp:83-102) around a
    device product y = A^T q (CSR / biclique kernels)."""
    import torch

    n = len(deg)
    d = torch.from_numpy(deg.astype(np.float64)).cuda()
    p = torch.full((n,), 1.0 / n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(p)
    it = 0
    for it in range(1, cfg.iterations + 1):
        q = torch.where(d > 0, p / d.clamp(min=1), torch.zeros_like(p))
        dm = p[d == 0].sum() if cfg.dangling == DanglingPolicy.UNIFORM else torch.zeros((), dtype=torch.float64,
                                                                                     device="cuda")
        multiply(q, y)
        nxt = cfg.alpha / n + (1.0 - cfg.alpha) * (y + dm / n)
        l1 = float((nxt - p).abs().sum())
        p = nxt
        if cfg.l1_tolerance is not None and l1 <= cfg.l1_tolerance:
            break
    return p.cpu().numpy(), it


def cmd_pagerank(a) -> None:
    import torch

    g = _graph(a.graph)
    cfg = PageRankConfig(alpha=a.alpha, iterations=a.iters, l1_tolerance=a.tol,
                         dangling=DanglingPolicy(a.dangling))
    deg = g.out_degrees()
    at = g.transpose()
    t0 = time.perf_counter()
    if a.kernel == "ref":
        dg = BvGraph(BvStream.encode(at, BvParams(window=a.window)), CreateOptions(device=a.device))
        res = pagerank(BvGpuKernel(dg), deg, cfg)
        ranks, it = res.ranks, res.iterations_run
    elif a.kernel == "csr":
        ro = torch.from_numpy(at.row_offsets.view(np.int64)).cuda()
        co = torch.from_numpy(at.columns.view(np.int32)).cuda()
        ranks, it = _power_iteration(lambda q, y: csr_matvec_device(ro, co, q, y), deg, cfg)
    else:
        cover = BicliqueCover.extract_greedy(at, min_gain=a.min_gain)
        k = BicliqueKernel(cover)
        ranks, it = _power_iteration(lambda q, y: k.multiply(q, y), deg, cfg)
    secs = time.perf_counter() - t0
    if a.out:
        np.savetxt(a.out, ranks, fmt="%.17g")
    top = np.argsort(-ranks)[:a.top]
    print(f"pagerank\tkernel={a.kernel}\tn={g.n}\tm={g.m}\titerations={it}\tsum={float(ranks.sum()):.15f}"
          f"\tseconds={secs:.4f}")
    for v in top:
        print(f"{int(v)}\t{ranks[v]:.12g}")


BENCH_HEADER = "name\tn\tm\tm_prime\tratio\tt\tt_prime\tS\tops\tops_prime\tlinf"


def cmd_bench(a) -> None:
    """run_bench: per graph, PageRank with the baseline CSR
    kernel and the compressed kernel, `reps` times each, median device time;
    a TSV row mirroring Table 1 (ratio m/m', t, t', S = t/t', adds per product,
    L-inf disagreement)."""
    print(BENCH_HEADER)
    cfg = PageRankConfig(alpha=a.alpha, iterations=a.iters, dangling=DanglingPolicy(a.dangling))
    for path in a.graphs:
        g = _graph(path)
        runs = [pagerank_equivalence_check(g, cfg, window=a.window, device=a.device) for _ in range(a.reps)]
        t = float(np.median([r.csr_seconds for r in runs]))
        tp = float(np.median([r.ref_seconds for r in runs]))
        r0 = runs[0]
        c = r0.compression
        print(f"{os.path.basename(path)}\t{g.n}\t{g.m}\t{c.m_prime}\t{c.ratio:.4f}\t{t:.6f}\t{tp:.6f}"
              f"\t{t / tp if tp else float('inf'):.3f}\t{r0.csr_adds}\t{r0.ref_adds}\t{max(r.linf for r in runs):.3e}")


def cmd_biclique(a) -> None:
    g = _graph(a.graph)
    cover = BicliqueCover.extract_greedy(g, min_gain=a.min_gain, max_rounds=a.max_rounds)
    if not cover.verify(g):
        raise RuntimeError("biclique cover does not cover the graph exactly")
    if a.out:
        cover.save(a.out)
    print(f"biclique-extract\tn={g.n}\tm={g.m}\tcompressed_size={cover.compressed_size}"
          f"\tratio={g.m / max(cover.compressed_size, 1):.4f}")


def parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="python -m paper_1708_07271_b200",
                                description="B200 compressed A.x / PageRank (arXiv:1708.07271)")
    sub = p.add_subparsers(dest="cmd", required=True)
    q = sub.add_parser("gen", help="seeded synthetic graph (copy model, social, Erdos-Renyi)")
    q.add_argument("--model", choices=["copy", "social", "er"], default="copy")
    q.add_argument("--n", type=int, required=True)
    q.add_argument("--degree", type=float, default=12.0)
    q.add_argument("--p-ref", type=float, default=0.7)
    q.add_argument("--p-copy", type=float, default=0.8)
    q.add_argument("--seed", type=int, default=0x170807271)
    q.add_argument("--window", type=int, default=7)
    q.add_argument("--out", required=True, help="edge-list text, or .cbv for a BV container")
    q.set_defaults(fn=cmd_gen)
    q = sub.add_parser("compress", help="edge list -> BV container (CBV1)")
    q.add_argument("graph")
    q.add_argument("--window", type=int, default=7)
    q.add_argument("--max-ref", type=int, default=3)
    q.add_argument("--n", type=int, default=None)
    q.add_argument("--out", required=True)
    q.set_defaults(fn=cmd_compress)
    q = sub.add_parser("stats", help="compression statistics (cmv::stats)")
    q.add_argument("graph")
    q.add_argument("--window", type=int, default=7)
    q.set_defaults(fn=cmd_stats)
    q = sub.add_parser("matvec", help="y = A x^T (gather) or y = x A (scatter) on the GPU")
    q.add_argument("graph")
    g = q.add_mutually_exclusive_group(required=True)
    g.add_argument("--vector", help="text file, one value per line")
    g.add_argument("--uniform", action="store_true", help="x uniform in [0, 1) (seeded)")
    q.add_argument("--seed", type=int, default=1)
    q.add_argument("--form", choices=["gather", "scatter", "left"], default="gather",
                   help="gather: A x^T; scatter: x A on A's compression; left: x A as (A^T) x (reference matvec_ref_left)")
    q.add_argument("--window", type=int, default=7)
    q.add_argument("--device", type=int, default=0)
    q.add_argument("--out", default=None)
    q.set_defaults(fn=cmd_matvec)
    q = sub.add_parser("pagerank", help="PageRank on the GPU")
    q.add_argument("graph")
    q.add_argument("--alpha", type=float, default=0.15)
    q.add_argument("--iters", type=int, default=50)
    q.add_argument("--tol", type=float, default=None)
    q.add_argument("--dangling", choices=["uniform", "drop"], default="uniform")
    q.add_argument("--kernel", choices=["csr", "ref", "biclique"], default="ref")
    q.add_argument("--window", type=int, default=7)
    q.add_argument("--min-gain", type=int, default=1)
    q.add_argument("--device", type=int, default=0)
    q.add_argument("--top", type=int, default=10)
    q.add_argument("--out", default=None)
    q.set_defaults(fn=cmd_pagerank)
    q = sub.add_parser("bench", help="Table-1 style TSV: CSR vs compressed PageRank")
    q.add_argument("graphs", nargs="+")
    q.add_argument("--reps", type=int, default=3)
    q.add_argument("--alpha", type=float, default=0.15)
    q.add_argument("--iters", type=int, default=50)
    q.add_argument("--dangling", choices=["uniform", "drop"], default="uniform")
    q.add_argument("--window", type=int, default=7)
    q.add_argument("--device", type=int, default=0)
    q.set_defaults(fn=cmd_bench)
    q = sub.add_parser("biclique-extract", help="greedy biclique cover (BCV1 text)")
    q.add_argument("graph")
    q.add_argument("--min-gain", type=int, default=1)
    q.add_argument("--max-rounds", type=int, default=UNBOUNDED_ROUNDS)
    q.add_argument("--out", default=None)
    q.set_defaults(fn=cmd_biclique)
    return p


def main(argv: Optional[List[str]] = None) -> int:
    a = parser().parse_args(argv)
    try:
        a.fn(a)
    except Exception as e:  # nonzero exit with a message on any error
        print(f"error: {type(e).__name__}: {e}", file=sys.stderr)
        return 1
    return 0
