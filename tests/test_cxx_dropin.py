"""The C++ drop-in: cmv::BvGpuKernel (include/cmv_b200/bv_gpu_kernel.hpp) is a
cmv::MatvecKernel -- the reference's own class when its headers are on the
include path (pagerank.hpp:27-34) -- and a reference-style pagerank written
against `const MatvecKernel&` runs unchanged on it."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"

TU = r"""
#include <type_traits>
#include "cmv_b200/bv_gpu_kernel.hpp"
static_assert(std::is_base_of_v<cmv::MatvecKernel, cmv::BvGpuKernel>);
static_assert(std::is_final_v<cmv::BvGpuKernel>);
static_assert(CMV_B200_REFERENCE_API == EXPECT_REF);
int main() { return 0; }
"""


def _compile(tmp_path, extra, expect_ref):
    src = tmp_path / "tu.cpp"
    src.write_text(TU.replace("EXPECT_REF", str(expect_ref)))
    cmd = ["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", f"-I{ROOT}/include"] + extra + [str(src)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_header_standalone(tmp_path):
    _compile(tmp_path, [], 0)


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present (GPU box)")
def test_header_against_reference_api(tmp_path):
    _compile(tmp_path, [f"-I{REF_INC}"], 1)


@pytest.mark.gpu
def test_dropin_example_runs(cuda, tmp_path):
    from oracle import pyoracle as O
    import paper_1708_07271_b200 as P

    exe = os.path.join(ROOT, "examples", "drop_in_pagerank")
    if not os.path.exists(exe):
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "examples")])
    n = 1 << 15
    out = tmp_path / "ranks.bin"
    r = subprocess.run([exe, str(n), str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    both = np.fromfile(out, dtype=np.float64).reshape(2, n)
    g = P.CsrGraph.copy_model(n, 24.0, 0.7, 0.8, seed=0x170807271 + 3)
    og = O.Csr.from_arrays(n, g.row_offsets, g.columns)
    want, _ = O.pagerank_csr(og.transpose(), og.out_degrees(), 0.15, 30)
    for p in both:
        assert np.max(np.abs(p - want) / want) <= 1e-12
