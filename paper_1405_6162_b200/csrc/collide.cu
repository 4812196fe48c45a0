// collide.cu -- the reference hot path on B200: D3Q19 binary BGK collision
// (reference pkg/src/latkit/kernels.py:89-125, _collision_range) and the
// 3-vector scale kernel (kernels.py:79-86, _scale_range).
//
// targetDP mapping: one CUDA thread per VVL-site chunk
// (TLP); the VVL sites of a chunk are consecutive in every SoA component, so
// they load as one 8*VVL-byte vector (ILP).  grid = ceil(nchunks / tpb).
//
// Register-resident single pass: all 2*19 values of a site stay in registers,
// one HBM read + one HBM write per value.
#include "ltk_common.cuh"

namespace ltk {

struct CollideArgs {
    double *f;
    double *g;
    long long padded, nsites, site_lo, nchunks;
    long long *err;
    double wv[Q];
    double cs2, tau_f, tau_g;
    // EXACT derived constants (same ops as the reference, hoisted -- CSE of
    // identical expressions is bitwise neutral)
    double c1;  // 2*cs2
    double c2;  // (2*cs2)*cs2
    // FAST derived constants
    double inv_tau_f, inv_tau_g, a1 /*1/cs2*/, a2 /*1/(2 cs2^2)*/, a3 /*1/(2 cs2)*/;
};

// Per-site moments accumulated component by component.
struct Site {
    double rho, jx, jy, jz, phi;
    double ux, uy, uz, t;  // t: EXACT usq/(2 cs2), FAST 1 - usq/(2 cs2)
    bool ok;
};

template <int I, class M>
__device__ __forceinline__ void accum_f(Site &s, double fi) {
    s.rho = M::add(s.rho, fi);
    if constexpr (cx(I) > 0) s.jx = M::add(s.jx, fi);
    if constexpr (cx(I) < 0) s.jx = M::sub(s.jx, fi);
    if constexpr (cy(I) > 0) s.jy = M::add(s.jy, fi);
    if constexpr (cy(I) < 0) s.jy = M::sub(s.jy, fi);
    if constexpr (cz(I) > 0) s.jz = M::add(s.jz, fi);
    if constexpr (cz(I) < 0) s.jz = M::sub(s.jz, fi);
}

template <int MODE>
__device__ __forceinline__ void finish_site(Site &s, const CollideArgs &a) {
    if constexpr (MODE == LTK_MODE_EXACT) {
        using M = Exact;
        const double rr = __drcp_rn(s.rho);  // RN(1/rho): three divisions by rho
        s.ux = div_rcp(s.jx, s.rho, rr);
        s.uy = div_rcp(s.jy, s.rho, rr);
        s.uz = div_rcp(s.jz, s.rho, rr);
        double usq = M::add(M::add(M::mul(s.ux, s.ux), M::mul(s.uy, s.uy)), M::mul(s.uz, s.uz));
        s.t = div_rcp(usq, a.c1, a.a3);
    } else {
        double inv = 1.0 / s.rho;
        s.ux = s.jx * inv;
        s.uy = s.jy * inv;
        s.uz = s.jz * inv;
        double usq = fma(s.ux, s.ux, fma(s.uy, s.uy, s.uz * s.uz));
        s.t = fma(-usq, a.a3, 1.0);
    }
}

// Relax component I of both distributions at one site.  EXACT: q = (u.c)/cs2
// and sq = ((u.c)(u.c))/((2 cs2) cs2) are passed in, because the opposite
// velocity reuses them: dot_c gives u.c_opp == -(u.c) exactly (RN is symmetric
// under negation), so (u.c_opp)/cs2 == -q and its square term == sq, and the
// bracket ((1 + q) + sq) - t is then bit-identical to the reference's.
// T1: bit 0 = tau_f == 1.0, bit 1 = tau_g == 1.0 (EXACT only).
template <int I, int T1>
__device__ __forceinline__ void relax_exact(double &f, double &g, double q, double sq,
                                            const Site &s, const CollideArgs &a) {
    using M = Exact;
    const double br = M::sub(M::add(M::add(1.0, q), sq), s.t);
    const double feq = M::mul(M::mul(a.wv[I], s.rho), br);
    const double geq = M::mul(M::mul(a.wv[I], s.phi), br);
    const double df = M::sub(f, feq), dg = M::sub(g, geq);
    if constexpr (T1 & 1) f = M::sub(f, df);  // x / 1.0 == x
    else f = M::sub(f, div_rcp(df, a.tau_f, a.inv_tau_f));
    if constexpr (T1 & 2) g = M::sub(g, dg);
    else g = M::sub(g, div_rcp(dg, a.tau_g, a.inv_tau_g));
}

template <int I>
__device__ __forceinline__ void relax_fast(double &f, double &g, const Site &s,
                                           const CollideArgs &a) {
    const double ud = dot_c<cx(I), cy(I), cz(I), Fast>(s.ux, s.uy, s.uz);
    const double br = fma(ud, fma(ud, a.a2, a.a1), s.t);
    const double feq = (a.wv[I] * s.rho) * br;
    const double geq = (a.wv[I] * s.phi) * br;
    f = fma(feq - f, a.inv_tau_f, f);
    g = fma(geq - g, a.inv_tau_g, g);
}

// Relax the pair {C, opp(C)} (C canonical) of site v.
template <int C, int MODE, int T1, int W>
__device__ __forceinline__ void relax_pair(double (&F)[Q][W], double (&G)[Q][W], int v,
                                           const Site &s, const CollideArgs &a) {
    constexpr int O = opp(C);
    if constexpr (MODE == LTK_MODE_EXACT) {
        using M = Exact;
        const double ud = dot_c<cx(C), cy(C), cz(C), M>(s.ux, s.uy, s.uz);
        const double q = div_rcp(ud, a.cs2, a.a1);
        const double sq = div_rcp(M::mul(ud, ud), a.c2, a.a2);
        relax_exact<C, T1>(F[C][v], G[C][v], q, sq, s, a);
        if constexpr (O != C) relax_exact<O, T1>(F[O][v], G[O][v], -q, sq, s, a);
    } else {
        relax_fast<C>(F[C][v], G[C][v], s, a);
        if constexpr (O != C) relax_fast<O>(F[O][v], G[O][v], s, a);
    }
}

template <int MODE>
struct Acc {
    using M = typename std::conditional<MODE == LTK_MODE_EXACT, Exact, Fast>::type;
};

// Register-resident collision of W (= 1 or 2) consecutive sites at base.
template <int W, int MODE, int T1>
__device__ __forceinline__ void collide_sites(double *__restrict__ f, double *__restrict__ g,
                                              long long base, const CollideArgs &a) {
    using M = typename Acc<MODE>::M;
    const long long P = a.padded;
    Site st[W];
#pragma unroll
    for (int v = 0; v < W; ++v) st[v] = Site{0.0, 0.0, 0.0, 0.0, 0.0, 0, 0, 0, 0, true};
    double F[Q][W], G[Q][W];
#pragma unroll
    for (int i = 0; i < Q; ++i) load_vec<W>(F[i], f + base + i * P);
#pragma unroll
    for (int i = 0; i < Q; ++i) load_vec<W>(G[i], g + base + i * P);
    static_for<0, Q>([&](auto I) {
#pragma unroll
        for (int v = 0; v < W; ++v) accum_f<I.value, M>(st[v], F[I.value][v]);
    });
#pragma unroll
    for (int v = 0; v < W; ++v) {
#pragma unroll
        for (int i = 0; i < Q; ++i) st[v].phi = M::add(st[v].phi, G[i][v]);
        if (st[v].rho <= 0.0) {  // kernels.py:106-109
            st[v].ok = false;
            if (base + v < a.nsites) flag_singular(a.err, base + v);
        } else {
            finish_site<MODE>(st[v], a);
        }
    }
    static_for<0, 10>([&](auto K) {
        constexpr int C = kCanon[K.value];
#pragma unroll
        for (int v = 0; v < W; ++v)
            if (st[v].ok) relax_pair<C, MODE, T1, W>(F, G, v, st[v], a);
    });
    // padding lanes (rho <= 0) are written back unchanged: bitwise untouched
#pragma unroll
    for (int i = 0; i < Q; ++i) store_vec<W>(f + base + i * P, F[i]);
#pragma unroll
    for (int i = 0; i < Q; ++i) store_vec<W>(g + base + i * P, G[i]);
}

// One thread per VVL-site chunk (TLP).  VVL <= 2 loads the chunk as 16-byte
// vectors in one register-resident pass; larger VVL walks the chunk's sites
// as 2-site vectors, so register use does not grow with VVL.
template <int VVL, int MODE, int T1>
__global__ void __launch_bounds__(256) k_collide(const CollideArgs a) {
    const long long chunk = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (chunk >= a.nchunks) return;
    const long long base = a.site_lo + chunk * VVL;
    if constexpr (VVL <= 2) {
        collide_sites<VVL, MODE, T1>(a.f, a.g, base, a);
    } else {
#pragma unroll 1
        for (int k = 0; k < VVL; k += 2) collide_sites<2, MODE, T1>(a.f, a.g, base + k, a);
    }
}

template <int VVL>
__global__ void __launch_bounds__(256) k_scale(double *field, long long padded,
                                               long long site_lo, long long nchunks, double a) {
    const long long chunk = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (chunk >= nchunks) return;
    double *p = field + site_lo + chunk * VVL;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        double t[VVL];
        load_vec<VVL>(t, p + c * padded);
#pragma unroll
        for (int v = 0; v < VVL; ++v) t[v] = __dmul_rn(a, t[v]);  // a*field, kernels.py:86
        store_vec<VVL>(p + c * padded, t);
    }
}

template <int MODE, int T1>
static int launch_collide(int vvl, int tpb, long long nchunks, const CollideArgs &a,
                          cudaStream_t st) {
    const unsigned grid = (unsigned)((nchunks + tpb - 1) / tpb);
    switch (vvl) {
        case 1: k_collide<1, MODE, T1><<<grid, tpb, 0, st>>>(a); break;
        case 2: k_collide<2, MODE, T1><<<grid, tpb, 0, st>>>(a); break;
        case 4: k_collide<4, MODE, T1><<<grid, tpb, 0, st>>>(a); break;
        case 8: k_collide<8, MODE, T1><<<grid, tpb, 0, st>>>(a); break;
        case 16: k_collide<16, MODE, T1><<<grid, tpb, 0, st>>>(a); break;
        default: return fail(LTK_ERR_PLAN, "unsupported vvl %d (1,2,4,8,16)", vvl);
    }
    LTK_CHECK_LAUNCH("k_collide");
    return LTK_OK;
}

static int check_range(int64_t chunk_lo, int64_t chunk_hi, int32_t vvl, int32_t tpb,
                       int64_t padded) {
    if (vvl != 1 && vvl != 2 && vvl != 4 && vvl != 8 && vvl != 16)
        return fail(LTK_ERR_PLAN, "unsupported vvl %d (1,2,4,8,16)", vvl);
    if (tpb < 32 || tpb > 256 || tpb % 32)
        return fail(LTK_ERR_PLAN, "tpb must be a multiple of 32 in [32, 256], got %d", tpb);
    if (chunk_lo < 0 || chunk_hi < chunk_lo || chunk_hi * (int64_t)vvl > padded)
        return fail(LTK_ERR_PLAN, "chunk range [%lld, %lld) x vvl %d exceeds padded %lld",
                    (long long)chunk_lo, (long long)chunk_hi, vvl, (long long)padded);
    if (padded % vvl)
        return fail(LTK_ERR_PLAN, "VVL %d does not divide padded extent %lld", vvl,
                    (long long)padded);
    return LTK_OK;
}

}  // namespace ltk

using namespace ltk;

extern "C" int ltk_collide(int64_t chunk_lo, int64_t chunk_hi, int32_t vvl, int32_t tpb,
                           double *f, double *g, int64_t padded, int64_t nsites,
                           const ltk_collision_params *p, void *stream) {
    int rc = check_range(chunk_lo, chunk_hi, vvl, tpb, padded);
    if (rc) return rc;
    if (!f || !g || !p) return fail(LTK_ERR_CONFIG, "null argument");
    if (chunk_hi == chunk_lo) return LTK_OK;
    if ((reinterpret_cast<uintptr_t>(f) | reinterpret_cast<uintptr_t>(g)) % 16)
        return fail(LTK_ERR_CONFIG, "field pointers must be 16-byte aligned");
    CollideArgs a;
    a.f = f;
    a.g = g;
    a.padded = padded;
    a.nsites = nsites;
    a.site_lo = chunk_lo * vvl;
    a.nchunks = chunk_hi - chunk_lo;
    cudaStream_t st = as_stream(stream);
    a.err = stream_word(st);
    if (!a.err) return fail(LTK_ERR_DEVICE, "stream error word unavailable");
    for (int i = 0; i < Q; ++i) a.wv[i] = p->wv[i];
    a.cs2 = p->cs2;
    a.tau_f = p->tau_f;
    a.tau_g = p->tau_g;
    a.c1 = 2.0 * p->cs2;
    a.c2 = a.c1 * p->cs2;
    a.inv_tau_f = 1.0 / p->tau_f;
    a.inv_tau_g = 1.0 / p->tau_g;
    a.a1 = 1.0 / p->cs2;
    a.a2 = 1.0 / a.c2;
    a.a3 = 1.0 / a.c1;
    if (p->mode == LTK_MODE_EXACT) {
        // x / 1.0 == x for every IEEE double: when tau is exactly 1 (the
        // reference default, model.py:48-49) the division is skipped, bitwise neutral
        switch ((p->tau_f == 1.0 ? 1 : 0) | (p->tau_g == 1.0 ? 2 : 0)) {
            case 0: return launch_collide<LTK_MODE_EXACT, 0>(vvl, tpb, a.nchunks, a, st);
            case 1: return launch_collide<LTK_MODE_EXACT, 1>(vvl, tpb, a.nchunks, a, st);
            case 2: return launch_collide<LTK_MODE_EXACT, 2>(vvl, tpb, a.nchunks, a, st);
            default: return launch_collide<LTK_MODE_EXACT, 3>(vvl, tpb, a.nchunks, a, st);
        }
    }
    if (p->mode == LTK_MODE_FAST) return launch_collide<LTK_MODE_FAST, 0>(vvl, tpb, a.nchunks, a, st);
    return fail(LTK_ERR_CONFIG, "unknown collision mode %d", p->mode);
}

extern "C" int ltk_scale(int64_t chunk_lo, int64_t chunk_hi, int32_t vvl, int32_t tpb,
                         double *field, int64_t padded, double a, void *stream) {
    int rc = check_range(chunk_lo, chunk_hi, vvl, tpb, padded);
    if (rc) return rc;
    if (chunk_hi == chunk_lo) return LTK_OK;
    const long long n = chunk_hi - chunk_lo;
    const unsigned grid = (unsigned)((n + tpb - 1) / tpb);
    cudaStream_t st = as_stream(stream);
    const long long lo = chunk_lo * vvl;
    switch (vvl) {
        case 1: k_scale<1><<<grid, tpb, 0, st>>>(field, padded, lo, n, a); break;
        case 2: k_scale<2><<<grid, tpb, 0, st>>>(field, padded, lo, n, a); break;
        case 4: k_scale<4><<<grid, tpb, 0, st>>>(field, padded, lo, n, a); break;
        case 8: k_scale<8><<<grid, tpb, 0, st>>>(field, padded, lo, n, a); break;
        default: k_scale<16><<<grid, tpb, 0, st>>>(field, padded, lo, n, a); break;
    }
    LTK_CHECK_LAUNCH("k_scale");
    return LTK_OK;
}

// Self-test of div_rcp (the EXACT division path) against the hardware
// division: out_rcp[k] = div_rcp(x, d, RN(1/d)), out_div[k] = __ddiv_rn(x, d).
__global__ void k_div_selftest(const double *x, const double *d, long long n, double *out_rcp,
                               double *out_div) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x) {
        const double r = __drcp_rn(d[k]);
        out_rcp[k] = ltk::div_rcp(x[k], d[k], r);
        out_div[k] = __ddiv_rn(x[k], d[k]);
    }
}

extern "C" int ltk_div_selftest(const double *x, const double *d, int64_t n, double *out_rcp,
                                double *out_div, void *stream) {
    if (n <= 0) return LTK_OK;
    const long long blocks = (n + 255) / 256;
    const unsigned g = (unsigned)(blocks < 148LL * 8 ? blocks : 148LL * 8);
    k_div_selftest<<<g, 256, 0, ltk::as_stream(stream)>>>(x, d, n, out_rcp, out_div);
    LTK_CHECK_LAUNCH("k_div_selftest");
    return LTK_OK;
}
