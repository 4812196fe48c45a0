// ltk_common.cuh -- shared helpers of libltk.so (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <type_traits>

#include "ltk.h"

namespace ltk {

// ---------------------------------------------------------------- errors
int fail(int status, const char *fmt, ...);
int cuda_fail(cudaError_t err, const char *what);
void count_launch(int n = 1);

#define LTK_CUDA(call)                                        \
    do {                                                      \
        cudaError_t e_ = (call);                              \
        if (e_ != cudaSuccess) return ltk::cuda_fail(e_, #call); \
    } while (0)

#define LTK_CHECK_LAUNCH(what)                                  \
    do {                                                        \
        cudaError_t e_ = cudaGetLastError();                    \
        if (e_ != cudaSuccess) return ltk::cuda_fail(e_, what); \
        ltk::count_launch();                                    \
    } while (0)

#define LTK_RC0(x)            \
    do {                      \
        int rc_ = (x);        \
        if (rc_) return rc_;  \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Device error words: 0 = no error, else LLONG_MAX - (lowest real site with
// rho <= 0), so the lowest site wins an atomicMax and a reset is a memset.
// Each CUDA stream has its own word (stream_word, runtime.cu) and each fluid
// engine owns one, so errors are reported to the caller whose kernels met
// them, never to another engine or device object sharing the GPU.
long long *stream_word(cudaStream_t st);
void release_stream_word(cudaStream_t st);
// Read the word on `st` (after the work that may set it), reset it, and
// return the site it records or -1.  Stream-ordered copies only.
int take_word(long long *word, cudaStream_t st, long long *site);

__device__ __forceinline__ void flag_singular(long long *word, long long site) {
    atomicMax(reinterpret_cast<unsigned long long *>(word),
              static_cast<unsigned long long>(0x7fffffffffffffffLL - site));
}

// ---------------------------------------------------------------- D3Q19
// Canonical ordering of reference model.py:21-34.
constexpr int Q = 19;
__host__ __device__ constexpr int cx(int i) {
    constexpr int t[Q] = {0, 1, -1, 0, 0, 0, 0, 1, 1, -1, -1, 1, 1, -1, -1, 0, 0, 0, 0};
    return t[i];
}
__host__ __device__ constexpr int cy(int i) {
    constexpr int t[Q] = {0, 0, 0, 1, -1, 0, 0, 1, -1, 1, -1, 0, 0, 0, 0, 1, 1, -1, -1};
    return t[i];
}
__host__ __device__ constexpr int cz(int i) {
    constexpr int t[Q] = {0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1};
    return t[i];
}

// Opposite velocity, c_opp(i) = -c_i (reference model.py:62-68 negation_index).
__host__ __device__ constexpr int opp(int i) {
    constexpr int t[Q] = {0, 2, 1, 4, 3, 6, 5, 10, 9, 8, 7, 14, 13, 12, 11, 18, 17, 16, 15};
    return t[i];
}

// The 10 canonical members of {i, opp(i)} (the smaller index; 0 is its own).
constexpr int kCanon[10] = {0, 1, 3, 5, 7, 8, 11, 12, 15, 16};

// Sum of ci*u over the nonzero velocity components, in x, y, z order.  The
// reference evaluates ((ux*cx + uy*cy) + uz*cz) with cx..cz in {0, +-1}:
// products by +-1 are exact and adding a +-0 product never changes a value
// (SURVEY.md Appendix B), so dropping zero terms is bitwise neutral.
template <int CX, int CY, int CZ, class M>
__device__ __forceinline__ double dot_c(double ux, double uy, double uz) {
    double acc = 0.0;
    bool first = true;
    if (CX != 0) { acc = CX > 0 ? ux : -ux; first = false; }
    if (CY != 0) {
        double t = CY > 0 ? uy : -uy;
        acc = first ? t : M::add(acc, t);
        first = false;
    }
    if (CZ != 0) {
        double t = CZ > 0 ? uz : -uz;
        acc = first ? t : M::add(acc, t);
        first = false;
    }
    return acc;
}

// Compile-time loop over the 19 velocities: f(std::integral_constant-like).
template <int I>
struct Int {
    static constexpr int value = I;
};
template <int I, int N, class F>
__device__ __forceinline__ void static_for(F &&f) {
    if constexpr (I < N) {
        f(Int<I>{});
        static_for<I + 1, N>(f);
    }
}

// ---------------------------------------------------------------- arithmetic
// EXACT: one IEEE round-to-nearest op per call, never contracted to FMA.
struct Exact {
    static constexpr bool exact = true;
    __device__ static __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    __device__ static __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    __device__ static __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    __device__ static __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
};

// Correctly rounded x / d from r = RN(1/d) (Markstein's theorem; Muller et
// al., Handbook of Floating-Point Arithmetic): q = RN(x r) is a faithful
// quotient because r has relative error < 2^-53, the remainder e = x - d q is
// exact in one FMA, and RN(q + e r) == RN(x / d) whenever nothing overflows or
// underflows.  So this is bitwise __ddiv_rn(x, d) for the lattice's operands
// in 3 dependent FP64 ops instead of the ~10-op, branchy division sequence.
// Edge cases (d > 0 finite everywhere here): the remainder is formed negated,
// en = q d - x, and the result as q - en r, so a zero x comes out with its own
// sign by plain IEEE arithmetic (x = -0: q = -0, en = +0, -0 + -0 = -0; x = +0:
// +0), and for every other x en = -e exactly, i.e. the same correctly rounded
// q + e r.  Only inf/NaN x (exponent all ones) need the pass-through, tested
// on the high word on the integer pipe: 3 FP64 instructions plus a LOP3, an
// ISETP and the 64-bit select per division.
__device__ __forceinline__ double div_rcp(double x, double d, double r) {
    const double q = __dmul_rn(x, r);
    const double en = __fma_rn(q, d, -x);
    const double res = __fma_rn(-en, r, q);
    const unsigned hi = (unsigned)__double2hiint(x);
    return (hi & 0x7ff00000u) == 0x7ff00000u ? x : res;
}

// FAST: plain operators (the compiler may contract to FMA).
struct Fast {
    static constexpr bool exact = false;
    __device__ static __forceinline__ double add(double a, double b) { return a + b; }
    __device__ static __forceinline__ double sub(double a, double b) { return a - b; }
    __device__ static __forceinline__ double mul(double a, double b) { return a * b; }
    __device__ static __forceinline__ double div(double a, double b) { return a / b; }
};

// Vector load/store of VVL consecutive doubles (VVL*8-byte aligned).
template <int VVL>
__device__ __forceinline__ void load_vec(double (&dst)[VVL], const double *p) {
    if constexpr (VVL == 1) {
        dst[0] = __ldg(p);
    } else {
#pragma unroll
        for (int k = 0; k < VVL; k += 2) {
            double2 t = __ldg(reinterpret_cast<const double2 *>(p + k));
            dst[k] = t.x;
            dst[k + 1] = t.y;
        }
    }
}

template <int VVL>
__device__ __forceinline__ void store_vec(double *p, const double (&src)[VVL]) {
    if constexpr (VVL == 1) {
        p[0] = src[0];
    } else {
#pragma unroll
        for (int k = 0; k < VVL; k += 2)
            *reinterpret_cast<double2 *>(p + k) = make_double2(src[k], src[k + 1]);
    }
}

}  // namespace ltk
