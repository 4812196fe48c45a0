// collide.cu -- the reference hot path on B200: D3Q19 binary BGK collision
// (reference pkg/src/latkit/kernels.py:89-125, _collision_range) and the
// 3-vector scale kernel (kernels.py:79-86, _scale_range).
//
// targetDP mapping: one CUDA thread per VVL-site chunk
// (TLP); the VVL sites of a chunk are consecutive in every SoA component, so
// they load as one 8*VVL-byte vector (ILP).  grid = ceil(nchunks / tpb).
//
// Two strategies, chosen by VVL at compile time:
//   VVL <= 2  register-resident: all 2*19*VVL values stay in registers, one
//             pass, one HBM read + one HBM write per value.
//   VVL >= 4  two-pass (the reference's own structure): pass 1 streams the
//             components to form the moments, pass 2 re-reads (L1/L2 hit),
//             relaxes and stores -- bounded register use at any VVL.
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
        s.ux = M::div(s.jx, s.rho);
        s.uy = M::div(s.jy, s.rho);
        s.uz = M::div(s.jz, s.rho);
        double usq = M::add(M::add(M::mul(s.ux, s.ux), M::mul(s.uy, s.uy)), M::mul(s.uz, s.uz));
        s.t = M::div(usq, a.c1);
    } else {
        double inv = 1.0 / s.rho;
        s.ux = s.jx * inv;
        s.uy = s.jy * inv;
        s.uz = s.jz * inv;
        double usq = fma(s.ux, s.ux, fma(s.uy, s.uy, s.uz * s.uz));
        s.t = fma(-usq, a.a3, 1.0);
    }
}

// Relax component I of both distributions at one site.
template <int I, int MODE>
__device__ __forceinline__ void relax(double &f, double &g, const Site &s, const CollideArgs &a) {
    if constexpr (MODE == LTK_MODE_EXACT) {
        using M = Exact;
        double ud = dot_c<cx(I), cy(I), cz(I), M>(s.ux, s.uy, s.uz);
        double br = M::sub(M::add(M::add(1.0, M::div(ud, a.cs2)), M::div(M::mul(ud, ud), a.c2)),
                           s.t);
        double feq = M::mul(M::mul(a.wv[I], s.rho), br);
        double geq = M::mul(M::mul(a.wv[I], s.phi), br);
        f = M::sub(f, M::div(M::sub(f, feq), a.tau_f));
        g = M::sub(g, M::div(M::sub(g, geq), a.tau_g));
    } else {
        double ud = dot_c<cx(I), cy(I), cz(I), Fast>(s.ux, s.uy, s.uz);
        double br = fma(ud, fma(ud, a.a2, a.a1), s.t);
        double feq = (a.wv[I] * s.rho) * br;
        double geq = (a.wv[I] * s.phi) * br;
        f = fma(feq - f, a.inv_tau_f, f);
        g = fma(geq - g, a.inv_tau_g, g);
    }
}

template <int MODE>
struct Acc {
    using M = typename std::conditional<MODE == LTK_MODE_EXACT, Exact, Fast>::type;
};

template <int VVL, int MODE>
__global__ void __launch_bounds__(256) k_collide(const CollideArgs a) {
    using M = typename Acc<MODE>::M;
    const long long chunk = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (chunk >= a.nchunks) return;
    const long long base = a.site_lo + chunk * VVL;
    double *__restrict__ f = a.f + base;
    double *__restrict__ g = a.g + base;
    const long long P = a.padded;

    Site st[VVL];
#pragma unroll
    for (int v = 0; v < VVL; ++v) st[v] = Site{0.0, 0.0, 0.0, 0.0, 0.0, 0, 0, 0, 0, true};

    if constexpr (VVL <= 2) {
        // ---------------- register-resident single pass
        double F[Q][VVL], G[Q][VVL];
#pragma unroll
        for (int i = 0; i < Q; ++i) load_vec<VVL>(F[i], f + i * P);
#pragma unroll
        for (int i = 0; i < Q; ++i) load_vec<VVL>(G[i], g + i * P);
        static_for<0, Q>([&](auto I) {
#pragma unroll
            for (int v = 0; v < VVL; ++v) accum_f<I.value, M>(st[v], F[I.value][v]);
        });
#pragma unroll
        for (int v = 0; v < VVL; ++v) {
#pragma unroll
            for (int i = 0; i < Q; ++i) st[v].phi = M::add(st[v].phi, G[i][v]);
            if (st[v].rho <= 0.0) {  // kernels.py:106-109
                st[v].ok = false;
                if (base + v < a.nsites) flag_singular(a.err, base + v);
            } else {
                finish_site<MODE>(st[v], a);
            }
        }
        static_for<0, Q>([&](auto I) {
#pragma unroll
            for (int v = 0; v < VVL; ++v) {
                if (st[v].ok) relax<I.value, MODE>(F[I.value][v], G[I.value][v], st[v], a);
            }
        });
#pragma unroll
        for (int i = 0; i < Q; ++i) store_vec<VVL>(f + i * P, F[i]);
#pragma unroll
        for (int i = 0; i < Q; ++i) store_vec<VVL>(g + i * P, G[i]);
    } else {
        // ---------------- two-pass: moments, then reload + relax + store
        static_for<0, Q>([&](auto I) {
            double t[VVL];
            load_vec<VVL>(t, f + I.value * P);
#pragma unroll
            for (int v = 0; v < VVL; ++v) accum_f<I.value, M>(st[v], t[v]);
        });
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            double t[VVL];
            load_vec<VVL>(t, g + i * P);
#pragma unroll
            for (int v = 0; v < VVL; ++v) st[v].phi = M::add(st[v].phi, t[v]);
        }
        bool any_ok = false;
#pragma unroll
        for (int v = 0; v < VVL; ++v) {
            if (st[v].rho <= 0.0) {
                st[v].ok = false;
                if (base + v < a.nsites) flag_singular(a.err, base + v);
            } else {
                finish_site<MODE>(st[v], a);
                any_ok = true;
            }
        }
        if (!any_ok) return;  // whole chunk is padding: untouched
        static_for<0, Q>([&](auto I) {
            double tf[VVL], tg[VVL];
            load_vec<VVL>(tf, f + I.value * P);
            load_vec<VVL>(tg, g + I.value * P);
#pragma unroll
            for (int v = 0; v < VVL; ++v)
                if (st[v].ok) relax<I.value, MODE>(tf[v], tg[v], st[v], a);
            store_vec<VVL>(f + I.value * P, tf);
            store_vec<VVL>(g + I.value * P, tg);
        });
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

template <int MODE>
static int launch_collide(int vvl, int tpb, long long nchunks, const CollideArgs &a,
                          cudaStream_t st) {
    const unsigned grid = (unsigned)((nchunks + tpb - 1) / tpb);
    switch (vvl) {
        case 1: k_collide<1, MODE><<<grid, tpb, 0, st>>>(a); break;
        case 2: k_collide<2, MODE><<<grid, tpb, 0, st>>>(a); break;
        case 4: k_collide<4, MODE><<<grid, tpb, 0, st>>>(a); break;
        case 8: k_collide<8, MODE><<<grid, tpb, 0, st>>>(a); break;
        case 16: k_collide<16, MODE><<<grid, tpb, 0, st>>>(a); break;
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
    a.err = singular_word();
    if (!a.err) return fail(LTK_ERR_DEVICE, "device error word unavailable");
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
    cudaStream_t st = as_stream(stream);
    if (p->mode == LTK_MODE_EXACT) return launch_collide<LTK_MODE_EXACT>(vvl, tpb, a.nchunks, a, st);
    if (p->mode == LTK_MODE_FAST) return launch_collide<LTK_MODE_FAST>(vvl, tpb, a.nchunks, a, st);
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
