// Run-time compilation of a model's dynamics (SURVEY.md §8 f row 2; expr.cpp:404-501).
//
// The bytecode program (gm_host.cpp Lowering) is turned into straight-line
// device code (one double per register, goto for the lazy ite), compiled by
// NVRTC together with the row-level kernels of gm_rowdev.cuh for sm_100a, and
// loaded with the CUDA runtime's library API. Same IEEE operations, same
// libdevice functions and --fmad=false as the ahead-of-time interpreter, so
// rows are bit-identical (tests/test_gpu_jit.py). NVRTC is loaded with dlopen:
// when it is absent or a compile fails the interpreter kernels are used.
#pragma once

#include "gm_host.hpp"

#include <string>

namespace gmj {

// Kernel handles (cudaKernel_t, usable as `const void*` function arguments of
// cudaLaunchKernel / cudaFuncSetAttribute / cudaOccupancy*).
struct Kernels {
    const void* build_ws[2] = {nullptr, nullptr}; // k_build_ws<false>, k_build_ws<true>
    const void* prologue = nullptr;              // k_prologue
    const void* ofa = nullptr;                   // k_expect_ofa_shape (kind 3)
    const void* ofa_packed = nullptr;            // k_expect_ofa_packed (kind 3)
    const void* ofa_group = nullptr;             // k_expect_ofa_group (kind 3)
    double compile_s = 0.0;
};

// CUDA source of `__device__ bool gm_dyn_jit(x, u, w, mu)` for program P.
std::string dynamics_source(const gmh::Program& P, int n);

enum Want { WANT_PROLOGUE = 1, WANT_BUILD_NOQS = 2, WANT_BUILD_QS = 4 };

// Compiled kernels for program P (cached per generated source; each kernel kind
// is its own NVRTC program, compiled on first use: ~2 s k_prologue, ~5 s
// k_build_ws), or nullptr with the reason in *why (NVRTC missing, compile or
// load failure, GM_JIT=0).
// `ctas`: resident CTAs per SM the build kernel is compiled for (its register cap,
// gmk::build_ctas).
const Kernels* kernels_for(const gmh::Program& P, int n, int m, int p, int want, std::string* why,
                           const std::string& shape = "", int ctas = 3);

// #defines that specialise the OFA consumer to a row shape (gm_ofa.cuh GM_OFA_SHAPE),
// or "" when the shape does not qualify; the compiled kernel for them (cached per
// process and on disk), nullptr with the reason in *why.
std::string ofa_shape_defines(const GmDev& D);
const void* ofa_kernel(const std::string& shape, double* compile_s, std::string* why,
                       const void** packed = nullptr, const void** group = nullptr);

// #defines that specialise the per-warp-Q build kernel (k_build_ws<true>) to one row
// shape (gm_rowdev.cuh GM_FILL_*), or "" when the shape does not qualify.
std::string shape_defines(const GmDev& D);

// NVRTC compile of one kernel kind (0 k_prologue, 1 k_build_ws<false>, 2
// k_build_ws<true>) without loading it: "" on success, else the compiler log.
// Needs no GPU (tests run it on the build host).
std::string compile_only(const gmh::Program& P, int n, int m, int p, int kind, double* seconds,
                         const std::string& shape = "", int ctas = 3);

} // namespace gmj
