"""Open problem families: a caller-defined __host__ __device__ family
(tests/cpp/user_family_test.cu, a shifted Rosenbrock with a cyclic coupling)
instantiates the GPU kernel through include/tronbatch_gpu/user_family.cuh in
its own translation unit; the same functions feed the reference's CPU
solve_batch (tron.hpp:28-36 BoundedProblem).  Every report bit-identical."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "user_family_test")


@pytest.mark.gpu
def test_user_family_matches_reference_solve_batch():
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/user_family_test not built (needs the reference headers at build time)")
    p = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "PASS: 0 of" in p.stdout


def test_user_family_header_compiles_for_sm100a(tmp_path):
    """The header-only path builds a caller's family for sm_100a without the
    reference headers (device entry point only) -- no GPU needed."""
    nvcc = "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    src = tmp_path / "fam.cu"
    src.write_text(r'''
#include "tronbatch_gpu/user_family.cuh"
struct Quad {
    static constexpr int kMaxDim = 8;
    __host__ __device__ static double f(const double* x, const double* p, int n) {
        double s = 0.0; for (int i = 0; i < n; ++i) s += (x[i] - p[i]) * (x[i] - p[i]); return s; }
    __host__ __device__ static double grad(const double* x, const double* p, int, int i) { return 2.0 * (x[i] - p[i]); }
    __host__ __device__ static double hess(const double*, const double*, int, int i, int j) { return i == j ? 2.0 : 0.0; }
};
template cudaError_t tronbatch::gpu::launch_user_batch<Quad>(int, int64_t, const double*, const double*, const double*,
    const double*, int64_t, int, const tb_tron_config&, double*, double*, double*, int32_t*, int32_t*, int64_t*,
    int64_t*, double*, cudaStream_t);
''')
    out = tmp_path / "fam.o"
    r = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "--fmad=false", "-std=c++17", "-c",
                        "-I", os.path.join(ROOT, "include"), str(src), "-o", str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    assert out.stat().st_size > 0
