// fluid_kernels.cuh -- device kernels of the full D3Q19 binary-fluid timestep
// (builder-defined extension).
//
// Slab layout: SoA, component stride cstride; storage plane
// zs = z + 1 holds owned plane z (zs = 0 and nzl + 1 are halo planes); site
// (x, y, zs) at zs*PL + y*nx + x with PL = nx*ny.  x is fastest, so a z-plane
// is one contiguous run of PL doubles per component (halo faces are plain
// contiguous NCCL buffers) and a warp touches 32 consecutive x.
//
// One timestep = k_phi -> k_mu -> k_collide_stream (pull scheme):
//   k_phi   phi(x) = sum_i g_i(x - c_i)                         [g pulled]
//   k_mu    mu = A phi + B phi^3 - kappa lap7(phi)               [phi stencil]
//   k_cs    pull f, g; phi again in registers; grad mu (central);
//           Guo-forced BGK for f, chemical-potential g_eq; aligned store.
// Halo images: a kernel that produces an owned boundary plane also stores it
// (phi, mu: the plane; f, g: the components that cross the face) straight into
// the halo plane that needs it -- the top plane into the bottom halo (zs = 0)
// of the slab above, the bottom plane into the top halo (zs = nzl+1) of the
// slab below.  One GPU, periodic z: both targets are this slab's own buffers,
// so a step needs no halo kernels.  z-slabs over NVLink (peer transport): the
// targets are the neighbours' buffers mapped with CUDA IPC, so the halo
// exchange is fused into the producing kernels as peer stores.  NCCL
// transport: no images (null targets); the engine exchanges faces instead.
#pragma once

#include "ltk_common.cuh"

namespace ltk {

struct FluidArgs {
    const double *f_in;
    const double *g_in;
    const double *mu;
    const double *phi_in;
    double *f_out;
    double *g_out;
    double *phi_out;
    double *mu_out;
    long long *err;
    int nx, ny, nzl, z_lo, nplanes;
    // halo image targets (nullptr = none): buffers of the slab above (up) /
    // below (dn); f/g point at the state being written (f_out/g_out side)
    double *img_f_up, *img_g_up, *img_f_dn, *img_g_dn;
    double *img_phi_up, *img_phi_dn, *img_mu_up, *img_mu_dn;
    long long PL, cstride;
    long long nthreads;   // threads of this launch
    long long nz_global, z0;  // for error-site reporting in host order
    double wv[Q];
    double lam[Q];
    double cs2, tau_f, tau_g, A, B, kappa, gamma;
    // derived (host-computed once, each the same IEEE expression as the oracle)
    double c1, c2, cs2sq, srcpre;                 // 2cs2, (2cs2)cs2, cs2*cs2, 1 - 0.5/tau_f
    double inv_tau_f, inv_tau_g, a1, a2, a3, inv_cs2, inv_cs2sq;  // FAST
};

// thread -> (x0, y, z) of a VVL-site row segment
struct Pos {
    int x0, y, z;
};

template <int VVL>
__device__ __forceinline__ bool thread_pos(const FluidArgs &a, Pos &p) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.nthreads) return false;
    const unsigned nxv = (unsigned)(a.nx / VVL);
    const unsigned tt = (unsigned)t;
    const unsigned row = tt / nxv;
    p.x0 = (int)(tt - row * nxv) * VVL;
    p.y = (int)(row % (unsigned)a.ny);
    p.z = a.z_lo + (int)(row / (unsigned)a.ny);
    return true;
}

__device__ __forceinline__ int wrapi(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

// Pull the VVL values of component I at sites (x0..x0+VVL-1, y, zs) from
// (x - cx, y - cy, zs - cz).  cx == 0 -> one aligned vector load.
template <int I, int VVL>
__device__ __forceinline__ void pull(double (&v)[VVL], const double *base, const FluidArgs &a,
                                     const Pos &p) {
    const int ys = wrapi(p.y - cy(I), a.ny);
    const double *row = base + (long long)I * a.cstride +
                        (long long)(p.z + 1 - cz(I)) * a.PL + (long long)ys * a.nx;
    if constexpr (cx(I) == 0) {
        load_vec<VVL>(v, row + p.x0);
    } else {
#pragma unroll
        for (int k = 0; k < VVL; ++k) v[k] = __ldg(row + wrapi(p.x0 + k - cx(I), a.nx));
    }
}

// ------------------------------------------------------------------ phi
template <int VVL>
__global__ void __launch_bounds__(256) k_phi(const FluidArgs a) {
    Pos p;
    if (!thread_pos<VVL>(a, p)) return;
    double phi[VVL];
#pragma unroll
    for (int k = 0; k < VVL; ++k) phi[k] = 0.0;
    static_for<0, Q>([&](auto I) {
        double v[VVL];
        pull<I.value, VVL>(v, a.g_in, a, p);
#pragma unroll
        for (int k = 0; k < VVL; ++k) phi[k] = __dadd_rn(phi[k], v[k]);
    });
    const long long off = (long long)p.y * a.nx + p.x0;
    store_vec<VVL>(a.phi_out + (long long)(p.z + 1) * a.PL + off, phi);
    // halo images for the mu stencil of the neighbouring slabs (or this one)
    bool img = false;
    if (p.z == 0 && a.img_phi_dn) {
        store_vec<VVL>(a.img_phi_dn + (long long)(a.nzl + 1) * a.PL + off, phi);
        img = true;
    }
    if (p.z == a.nzl - 1 && a.img_phi_up) {
        store_vec<VVL>(a.img_phi_up + off, phi);
        img = true;
    }
    if (img) __threadfence_system();  // peer images visible before the progress signal
}

// ------------------------------------------------------------------ mu
// mu = (A phi + B phi^3) - kappa lap, lap = (((((phi(x+1) + phi(x-1)) + phi(y+1))
//      + phi(y-1)) + phi(z+1)) + phi(z-1)) - 6 phi   (oracle orc_mu op order)
template <int VVL>
__global__ void __launch_bounds__(256) k_mu(const FluidArgs a) {
    Pos p;
    if (!thread_pos<VVL>(a, p)) return;
    const double *c = a.phi_in + (long long)(p.z + 1) * a.PL;
    const int yp = wrapi(p.y + 1, a.ny), ym = wrapi(p.y - 1, a.ny);
    double mu[VVL];
#pragma unroll
    for (int k = 0; k < VVL; ++k) {
        const int x = p.x0 + k;
        const int xp = wrapi(x + 1, a.nx), xm = wrapi(x - 1, a.nx);
        const double ph = __ldg(c + (long long)p.y * a.nx + x);
        double s = __ldg(c + (long long)p.y * a.nx + xp);
        s = __dadd_rn(s, __ldg(c + (long long)p.y * a.nx + xm));
        s = __dadd_rn(s, __ldg(c + (long long)yp * a.nx + x));
        s = __dadd_rn(s, __ldg(c + (long long)ym * a.nx + x));
        s = __dadd_rn(s, __ldg(c + a.PL + (long long)p.y * a.nx + x));
        s = __dadd_rn(s, __ldg(c - a.PL + (long long)p.y * a.nx + x));
        const double lap = __dsub_rn(s, __dmul_rn(6.0, ph));
        const double p3 = __dmul_rn(__dmul_rn(ph, ph), ph);
        mu[k] = __dsub_rn(__dadd_rn(__dmul_rn(a.A, ph), __dmul_rn(a.B, p3)),
                          __dmul_rn(a.kappa, lap));
    }
    const long long off = (long long)p.y * a.nx + p.x0;
    store_vec<VVL>(a.mu_out + (long long)(p.z + 1) * a.PL + off, mu);
    bool img = false;
    if (p.z == 0 && a.img_mu_dn) {
        store_vec<VVL>(a.img_mu_dn + (long long)(a.nzl + 1) * a.PL + off, mu);
        img = true;
    }
    if (p.z == a.nzl - 1 && a.img_mu_up) {
        store_vec<VVL>(a.img_mu_up + off, mu);
        img = true;
    }
    if (img) __threadfence_system();
}

// ------------------------------------------------------------------ collide-stream
struct FSite {
    double rho, jx, jy, jz, phi, mu;
    double Fx, Fy, Fz, ux, uy, uz, t, uF, psi;
};

template <int I, class M>
__device__ __forceinline__ void faccum(FSite &s, double fi) {
    s.rho = M::add(s.rho, fi);
    if constexpr (cx(I) > 0) s.jx = M::add(s.jx, fi);
    if constexpr (cx(I) < 0) s.jx = M::sub(s.jx, fi);
    if constexpr (cy(I) > 0) s.jy = M::add(s.jy, fi);
    if constexpr (cy(I) < 0) s.jy = M::sub(s.jy, fi);
    if constexpr (cz(I) > 0) s.jz = M::add(s.jz, fi);
    if constexpr (cz(I) < 0) s.jz = M::sub(s.jz, fi);
}

// Site-wide quantities after the moments (oracle collide_site op order).
template <int MODE, int PHYS>
__device__ __forceinline__ void fsite_finish(FSite &s, double gmx, double gmy, double gmz,
                                             const FluidArgs &a) {
    using M = Exact;
    if constexpr (MODE == LTK_MODE_EXACT) {
        if constexpr (PHYS == 1) {
            s.Fx = -M::mul(s.phi, gmx);
            s.Fy = -M::mul(s.phi, gmy);
            s.Fz = -M::mul(s.phi, gmz);
            s.ux = M::div(M::add(s.jx, M::mul(0.5, s.Fx)), s.rho);
            s.uy = M::div(M::add(s.jy, M::mul(0.5, s.Fy)), s.rho);
            s.uz = M::div(M::add(s.jz, M::mul(0.5, s.Fz)), s.rho);
            s.uF = M::add(M::add(M::mul(s.ux, s.Fx), M::mul(s.uy, s.Fy)), M::mul(s.uz, s.Fz));
            s.psi = M::sub(M::mul(a.gamma, s.mu), M::mul(s.phi, a.cs2));
        } else {
            s.ux = M::div(s.jx, s.rho);
            s.uy = M::div(s.jy, s.rho);
            s.uz = M::div(s.jz, s.rho);
        }
        const double usq =
            M::add(M::add(M::mul(s.ux, s.ux), M::mul(s.uy, s.uy)), M::mul(s.uz, s.uz));
        s.t = M::div(usq, a.c1);
    } else {
        const double inv = 1.0 / s.rho;
        if constexpr (PHYS == 1) {
            s.Fx = -(s.phi * gmx);
            s.Fy = -(s.phi * gmy);
            s.Fz = -(s.phi * gmz);
            s.ux = fma(0.5, s.Fx, s.jx) * inv;
            s.uy = fma(0.5, s.Fy, s.jy) * inv;
            s.uz = fma(0.5, s.Fz, s.jz) * inv;
            s.uF = fma(s.ux, s.Fx, fma(s.uy, s.Fy, s.uz * s.Fz));
            s.psi = fma(a.gamma, s.mu, -(s.phi * a.cs2));
        } else {
            s.ux = s.jx * inv;
            s.uy = s.jy * inv;
            s.uz = s.jz * inv;
        }
        const double usq = fma(s.ux, s.ux, fma(s.uy, s.uy, s.uz * s.uz));
        s.t = fma(-usq, a.a3, 1.0);
    }
}

// T1 (EXACT): bit 0 = tau_f == 1.0, bit 1 = tau_g == 1.0 -> x / 1.0 == x, skip it.
// EXACT: q = (u.c)/cs2 and sq = ((u.c)(u.c))/((2cs2)cs2) come from the pair's
// canonical velocity; the opposite velocity gets -q and sq, which leaves the
// bracket ((1 + q) + sq) - t bit-identical (see collide.cu relax_exact).
template <int I, int MODE, int PHYS, int T1>
__device__ __forceinline__ void frelax(double &f, double &g, double q, double sq, const FSite &s,
                                       const FluidArgs &a) {
    if constexpr (MODE == LTK_MODE_EXACT) {
        using M = Exact;
        const double br = M::sub(M::add(M::add(1.0, q), sq), s.t);
        const double feq = M::mul(M::mul(a.wv[I], s.rho), br);
        double geq = M::mul(M::mul(a.wv[I], s.phi), br);
        const double df = M::sub(f, feq);
        double fn;
        if constexpr (T1 & 1) fn = M::sub(f, df);
        else fn = M::sub(f, M::div(df, a.tau_f));
        if constexpr (PHYS == 1) {
            const double ud = dot_c<cx(I), cy(I), cz(I), M>(s.ux, s.uy, s.uz);
            const double cF = dot_c<cx(I), cy(I), cz(I), M>(s.Fx, s.Fy, s.Fz);
            const double src =
                M::mul(M::mul(a.srcpre, a.wv[I]),
                       M::add(M::div(M::sub(cF, s.uF), a.cs2), M::div(M::mul(ud, cF), a.cs2sq)));
            fn = M::add(fn, src);
            geq = M::add(geq, M::mul(a.lam[I], s.psi));
        }
        f = fn;
        const double dg = M::sub(g, geq);
        if constexpr (T1 & 2) g = M::sub(g, dg);
        else g = M::sub(g, M::div(dg, a.tau_g));
    } else {
        const double ud = dot_c<cx(I), cy(I), cz(I), Fast>(s.ux, s.uy, s.uz);
        const double br = fma(ud, fma(ud, a.a2, a.a1), s.t);
        const double feq = (a.wv[I] * s.rho) * br;
        double geq = (a.wv[I] * s.phi) * br;
        double fn = fma(feq - f, a.inv_tau_f, f);
        if constexpr (PHYS == 1) {
            const double cF = dot_c<cx(I), cy(I), cz(I), Fast>(s.Fx, s.Fy, s.Fz);
            const double src = (a.srcpre * a.wv[I]) *
                               fma(ud * cF, a.inv_cs2sq, (cF - s.uF) * a.inv_cs2);
            fn += src;
            geq = fma(a.lam[I], s.psi, geq);
        }
        f = fn;
        g = fma(geq - g, a.inv_tau_g, g);
    }
}

// Relax the pair {C, opp(C)} (C canonical) of lane k.
template <int C, int MODE, int PHYS, int T1, int VVL>
__device__ __forceinline__ void frelax_pair(double (&F)[Q][VVL], double (&G)[Q][VVL], int k,
                                            const FSite &s, const FluidArgs &a) {
    constexpr int O = opp(C);
    double q = 0.0, sq = 0.0;
    if constexpr (MODE == LTK_MODE_EXACT) {
        using M = Exact;
        const double ud = dot_c<cx(C), cy(C), cz(C), M>(s.ux, s.uy, s.uz);
        q = M::div(ud, a.cs2);
        sq = M::div(M::mul(ud, ud), a.c2);
    }
    frelax<C, MODE, PHYS, T1>(F[C][k], G[C][k], q, sq, s, a);
    if constexpr (O != C) frelax<O, MODE, PHYS, T1>(F[O][k], G[O][k], -q, sq, s, a);
}

template <int VVL, int MODE, int PHYS, int T1>
__global__ void __launch_bounds__(128, VVL == 1 ? 4 : 1) k_collide_stream(const FluidArgs a) {
    using M = typename std::conditional<MODE == LTK_MODE_EXACT, Exact, Fast>::type;
    Pos p;
    if (!thread_pos<VVL>(a, p)) return;

    double F[Q][VVL], G[Q][VVL];
    static_for<0, Q>([&](auto I) { pull<I.value, VVL>(F[I.value], a.f_in, a, p); });
    static_for<0, Q>([&](auto I) { pull<I.value, VVL>(G[I.value], a.g_in, a, p); });

    FSite st[VVL];
#pragma unroll
    for (int k = 0; k < VVL; ++k) st[k] = FSite{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0,
                                                0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    static_for<0, Q>([&](auto I) {
#pragma unroll
        for (int k = 0; k < VVL; ++k) faccum<I.value, M>(st[k], F[I.value][k]);
    });
    bool ok[VVL];
    const double *mc = a.mu + (long long)(p.z + 1) * a.PL;
    const int yp = wrapi(p.y + 1, a.ny), ym = wrapi(p.y - 1, a.ny);
#pragma unroll
    for (int k = 0; k < VVL; ++k) {
#pragma unroll
        for (int i = 0; i < Q; ++i) st[k].phi = M::add(st[k].phi, G[i][k]);
        double gmx = 0.0, gmy = 0.0, gmz = 0.0;
        if constexpr (PHYS == 1) {
            const int x = p.x0 + k;
            const long long r = (long long)p.y * a.nx;
            st[k].mu = __ldg(mc + r + x);
            gmx = Exact::mul(Exact::sub(__ldg(mc + r + wrapi(x + 1, a.nx)),
                                        __ldg(mc + r + wrapi(x - 1, a.nx))), 0.5);
            gmy = Exact::mul(Exact::sub(__ldg(mc + (long long)yp * a.nx + x),
                                        __ldg(mc + (long long)ym * a.nx + x)), 0.5);
            gmz = Exact::mul(Exact::sub(__ldg(mc + a.PL + r + x), __ldg(mc - a.PL + r + x)), 0.5);
        }
        ok[k] = !(st[k].rho <= 0.0);
        if (ok[k]) {
            fsite_finish<MODE, PHYS>(st[k], gmx, gmy, gmz, a);
        } else {  // leave the streamed values; report the site in host order
            const long long zg = a.z0 + p.z;
            const long long site = ((long long)(p.x0 + k) * a.ny + p.y) * a.nz_global + zg;
            flag_singular(a.err, site);
        }
    }
    static_for<0, 10>([&](auto K) {
        constexpr int C = kCanon[K.value];
#pragma unroll
        for (int k = 0; k < VVL; ++k)
            if (ok[k]) frelax_pair<C, MODE, PHYS, T1, VVL>(F, G, k, st[k], a);
    });

    const long long off = (long long)p.y * a.nx + p.x0;
    const long long o = (long long)(p.z + 1) * a.PL + off;
    static_for<0, Q>([&](auto I) {
        store_vec<VVL>(a.f_out + I.value * a.cstride + o, F[I.value]);
        store_vec<VVL>(a.g_out + I.value * a.cstride + o, G[I.value]);
        // halo images of the components that cross the z faces
        if constexpr (cz(I.value) < 0) {
            if (p.z == 0 && a.img_f_dn) {
                const long long h = (long long)(a.nzl + 1) * a.PL + off;
                store_vec<VVL>(a.img_f_dn + I.value * a.cstride + h, F[I.value]);
                store_vec<VVL>(a.img_g_dn + I.value * a.cstride + h, G[I.value]);
            }
        }
        if constexpr (cz(I.value) > 0) {
            if (p.z == a.nzl - 1 && a.img_f_up) {
                store_vec<VVL>(a.img_f_up + I.value * a.cstride + off, F[I.value]);
                store_vec<VVL>(a.img_g_up + I.value * a.cstride + off, G[I.value]);
            }
        }
    });
    if ((p.z == 0 && a.img_f_dn) || (p.z == a.nzl - 1 && a.img_f_up))
        __threadfence_system();  // peer images visible before the progress signal
}

}  // namespace ltk
