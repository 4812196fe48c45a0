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
    double *phi_next;  // k_cs_phi: phi of the state being written
    // physics 2 (stress form): p_iso, d_x phi, d_y phi, d_z phi, slab layout like
    // mu, at aux + k * astride; written by the mu kernels, read by collide-stream
    double *aux, *img_aux_up, *img_aux_dn;
    long long astride;
    long long *err;
    int nx, ny, nzl, z_lo, nplanes;
    // halo image targets (nullptr = none): buffers of the slab above (up) /
    // below (dn); f/g point at the state being written (f_out/g_out side)
    double *img_f_up, *img_g_up, *img_f_dn, *img_g_dn;
    double *img_phi_up, *img_phi_dn, *img_mu_up, *img_mu_dn;
    long long PL, cstride;
    // f/g element (component i, storage plane zs, row y, x) at i*SI + zs*SZ + y*SY + x:
    // SoA (SI, SZ, SY) = (cstride, PL, nx); row-blocked (nx, ny*Q*nx, Q*nx)
    long long SI, SZ, SY;
    long long nthreads;   // threads of this launch
    long long nz_global, z0;  // for error-site reporting in host order
    // fused collide-stream + next-state phi (k_cs_phi); see that kernel
    unsigned long long *sync;  // [0] ticket, [1 + z] plane z sites done (cumulative)
    long long tpp;             // threads per plane (ny * nx / VVL)
    int phi_lo, phi_hi;        // phi planes of the next state formed in-kernel
    unsigned lag_ctas;         // phi work of CTA b is the phi thread range of CTA b - lag_ctas
    unsigned ncta_cs, ncta;    // CTAs with collide work / all CTAs
    double wv[Q];
    double lam[Q];
    double sw[Q];  // srcpre * wv[i] (host, the same RN product the oracle forms per site)
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
__device__ __forceinline__ void pos_of(const FluidArgs &a, unsigned tt, int z_lo, Pos &p) {
    const unsigned nxv = (unsigned)(a.nx / VVL);
    const unsigned row = tt / nxv;
    p.x0 = (int)(tt - row * nxv) * VVL;
    p.y = (int)(row % (unsigned)a.ny);
    p.z = z_lo + (int)(row / (unsigned)a.ny);
}

template <int VVL>
__device__ __forceinline__ bool thread_pos(const FluidArgs &a, Pos &p) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.nthreads) return false;
    pos_of<VVL>(a, (unsigned)t, a.z_lo, p);
    return true;
}

// Load flavours of pull(): plain read-only (__ldg), read-only with an L2
// policy (the fused kernel's input state), L2-only with a policy (state
// written earlier in the same launch).
enum { kLdg = 0, kLdNc = 1, kLdCg = 2 };

__device__ __forceinline__ int wrapi(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

// Pull the VVL values of component I at sites (x0..x0+VVL-1, y, zs) from
// (x - cx, y - cy, zs - cz).  cx == 0 -> one aligned vector load.
template <int I, int VVL, int LD = kLdg>
__device__ __forceinline__ void pull(double (&v)[VVL], const double *base, const FluidArgs &a,
                                     const Pos &p, uint64_t pol = 0) {
    const int ys = wrapi(p.y - cy(I), a.ny);
    const double *row = base + (long long)I * a.SI + (long long)(p.z + 1 - cz(I)) * a.SZ +
                        (long long)ys * a.SY;
    if constexpr (cx(I) == 0) {
        if constexpr (LD == kLdg) load_vec<VVL>(v, row + p.x0);
        else if constexpr (LD == kLdNc) load_vec_nc<VVL>(v, row + p.x0, pol);
        else load_vec_cg<VVL>(v, row + p.x0, pol);
    } else {
#pragma unroll
        for (int k = 0; k < VVL; ++k) {
            const double *q = row + wrapi(p.x0 + k - cx(I), a.nx);
            if constexpr (LD == kLdg) v[k] = __ldg(q);
            else if constexpr (LD == kLdNc) v[k] = ld_nc_pol(q, pol);
            else v[k] = ld_cg_pol(q, pol);
        }
    }
}

// ------------------------------------------------------------------ phi
template <int VVL, int LD, bool IMG = true>
__device__ __forceinline__ void phi_site(const FluidArgs &a, const Pos &p, const double *g,
                                         double *out, uint64_t pol) {
    double phi[VVL];
#pragma unroll
    for (int k = 0; k < VVL; ++k) phi[k] = 0.0;
    double v[Q][VVL];  // all loads issued before the first add
    static_for<0, Q>([&](auto I) { pull<I.value, VVL, LD>(v[I.value], g, a, p, pol); });
    static_for<0, Q>([&](auto I) {
#pragma unroll
        for (int k = 0; k < VVL; ++k) phi[k] = __dadd_rn(phi[k], v[I.value][k]);
    });
    const long long off = (long long)p.y * a.nx + p.x0;
    store_vec<VVL>(out + (long long)(p.z + 1) * a.PL + off, phi);
    if constexpr (!IMG) return;
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

template <int VVL>
__global__ void __launch_bounds__(256) k_phi(const FluidArgs a) {
    Pos p;
    if (!thread_pos<VVL>(a, p)) return;
    phi_site<VVL, kLdg>(a, p, a.g_in, a.phi_out, 0);
}

// ------------------------------------------------------------------ mu
// physics 2 side outputs of the mu kernels at storage offset o = zs*PL + off:
// p_iso and the central gradient of phi (oracle orc_stress op order), plus
// their halo images for the boundary planes (like mu's).
__device__ __forceinline__ void stress_store(const FluidArgs &a, int z, long long off, double ph,
                                             double mu, double xp, double xm, double yp, double ym,
                                             double zp, double zm) {
    using M = Exact;
    const double gx = M::mul(M::sub(xp, xm), 0.5);
    const double gy = M::mul(M::sub(yp, ym), 0.5);
    const double gz = M::mul(M::sub(zp, zm), 0.5);
    const double gsq = M::add(M::add(M::mul(gx, gx), M::mul(gy, gy)), M::mul(gz, gz));
    const double pp = M::mul(ph, ph);
    const double fb = M::add(M::mul(M::mul(0.5, a.A), pp), M::mul(M::mul(0.25, a.B), M::mul(pp, pp)));
    const double piso = M::sub(M::sub(M::mul(ph, mu), fb), M::mul(M::mul(0.5, a.kappa), gsq));
    const double v[4] = {piso, gx, gy, gz};
    const long long o = (long long)(z + 1) * a.PL + off;
#pragma unroll
    for (int k = 0; k < 4; ++k) a.aux[k * a.astride + o] = v[k];
    if (z == 0 && a.img_aux_dn) {
        const long long h = (long long)(a.nzl + 1) * a.PL + off;
#pragma unroll
        for (int k = 0; k < 4; ++k) a.img_aux_dn[k * a.astride + h] = v[k];
    }
    if (z == a.nzl - 1 && a.img_aux_up) {
#pragma unroll
        for (int k = 0; k < 4; ++k) a.img_aux_up[k * a.astride + off] = v[k];
    }
}

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
        if (a.aux)
            stress_store(a, p.z, (long long)p.y * a.nx + x, ph, mu[k],
                         __ldg(c + (long long)p.y * a.nx + xp), __ldg(c + (long long)p.y * a.nx + xm),
                         __ldg(c + (long long)yp * a.nx + x), __ldg(c + (long long)ym * a.nx + x),
                         __ldg(c + a.PL + (long long)p.y * a.nx + x),
                         __ldg(c - a.PL + (long long)p.y * a.nx + x));
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
        if constexpr (PHYS >= 1) {
            if constexpr (PHYS == 1) {
                s.Fx = -M::mul(s.phi, gmx);
                s.Fy = -M::mul(s.phi, gmy);
                s.Fz = -M::mul(s.phi, gmz);
            } else {  // the stress-divergence force itself
                s.Fx = gmx;
                s.Fy = gmy;
                s.Fz = gmz;
            }
            const double rr = __drcp_rn(s.rho);  // RN(1/rho): three divisions by rho
            s.ux = div_rcp(M::add(s.jx, M::mul(0.5, s.Fx)), s.rho, rr);
            s.uy = div_rcp(M::add(s.jy, M::mul(0.5, s.Fy)), s.rho, rr);
            s.uz = div_rcp(M::add(s.jz, M::mul(0.5, s.Fz)), s.rho, rr);
            s.uF = M::add(M::add(M::mul(s.ux, s.Fx), M::mul(s.uy, s.Fy)), M::mul(s.uz, s.Fz));
            s.psi = M::sub(M::mul(a.gamma, s.mu), M::mul(s.phi, a.cs2));
        } else {
            const double rr = __drcp_rn(s.rho);
            s.ux = div_rcp(s.jx, s.rho, rr);
            s.uy = div_rcp(s.jy, s.rho, rr);
            s.uz = div_rcp(s.jz, s.rho, rr);
        }
        const double usq =
            M::add(M::add(M::mul(s.ux, s.ux), M::mul(s.uy, s.uy)), M::mul(s.uz, s.uz));
        s.t = div_rcp(usq, a.c1, a.a3);
    } else {
        const double inv = 1.0 / s.rho;
        if constexpr (PHYS >= 1) {
            if constexpr (PHYS == 1) {
                s.Fx = -(s.phi * gmx);
                s.Fy = -(s.phi * gmy);
                s.Fz = -(s.phi * gmz);
            } else {
                s.Fx = gmx;
                s.Fy = gmy;
                s.Fz = gmz;
            }
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
__device__ __forceinline__ void frelax(double &f, double &g, double q, double sq, double s2,
                                       const FSite &s, const FluidArgs &a) {
    if constexpr (MODE == LTK_MODE_EXACT) {
        using M = Exact;
        const double br = M::sub(M::add(M::add(1.0, q), sq), s.t);
        const double feq = M::mul(M::mul(a.wv[I], s.rho), br);
        double geq = M::mul(M::mul(a.wv[I], s.phi), br);
        const double df = M::sub(f, feq);
        double fn;
        if constexpr (T1 & 1) fn = M::sub(f, df);
        else fn = M::sub(f, div_rcp(df, a.tau_f, a.inv_tau_f));
        if constexpr (PHYS >= 1) {
            // s2 = ((u.c)(F.c))/(cs2 cs2) from the pair (frelax_pair): the opposite
            // velocity's factors are both negated exactly, so the product is equal
            const double cF = dot_c<cx(I), cy(I), cz(I), M>(s.Fx, s.Fy, s.Fz);
            const double src = M::mul(a.sw[I],
                                      M::add(div_rcp(M::sub(cF, s.uF), a.cs2, a.inv_cs2), s2));
            fn = M::add(fn, src);
            geq = M::add(geq, M::mul(a.lam[I], s.psi));
        }
        f = fn;
        const double dg = M::sub(g, geq);
        if constexpr (T1 & 2) g = M::sub(g, dg);
        else g = M::sub(g, div_rcp(dg, a.tau_g, a.inv_tau_g));
    } else {
        const double ud = dot_c<cx(I), cy(I), cz(I), Fast>(s.ux, s.uy, s.uz);
        const double br = fma(ud, fma(ud, a.a2, a.a1), s.t);
        const double feq = (a.wv[I] * s.rho) * br;
        double geq = (a.wv[I] * s.phi) * br;
        double fn = fma(feq - f, a.inv_tau_f, f);
        if constexpr (PHYS >= 1) {
            const double cF = dot_c<cx(I), cy(I), cz(I), Fast>(s.Fx, s.Fy, s.Fz);
            const double src = a.sw[I] *
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
    double q = 0.0, sq = 0.0, s2 = 0.0;
    if constexpr (MODE == LTK_MODE_EXACT) {
        using M = Exact;
        const double ud = dot_c<cx(C), cy(C), cz(C), M>(s.ux, s.uy, s.uz);
        q = div_rcp(ud, a.cs2, a.a1);
        sq = div_rcp(M::mul(ud, ud), a.c2, a.a2);
        if constexpr (PHYS >= 1) {
            const double cF = dot_c<cx(C), cy(C), cz(C), M>(s.Fx, s.Fy, s.Fz);
            s2 = div_rcp(M::mul(ud, cF), a.cs2sq, a.inv_cs2sq);
        }
    }
    frelax<C, MODE, PHYS, T1>(F[C][k], G[C][k], q, sq, s2, s, a);
    if constexpr (O != C) frelax<O, MODE, PHYS, T1>(F[O][k], G[O][k], -q, sq, s2, s, a);
}

// One VVL-site chunk of the pull + forced collision.  HINT bit 0: the input
// state is read with L2 evict-first (each value is pulled once); bit 1: f' is
// stored evict-first and g' evict-last, so g' stays in L2 until k_cs_phi's
// lagged phi re-reads it a few planes later.
template <int VVL, int HINT>
__device__ __forceinline__ void cs_load(const FluidArgs &a, const Pos &p, double (&F)[Q][VVL],
                                        double (&G)[Q][VVL]) {
    const uint64_t pol = (HINT & 1) ? l2_evict_first() : 0;
    constexpr int LD = (HINT & 1) ? kLdNc : kLdg;
    static_for<0, Q>([&](auto I) { pull<I.value, VVL, LD>(F[I.value], a.f_in, a, p, pol); });
    static_for<0, Q>([&](auto I) { pull<I.value, VVL, LD>(G[I.value], a.g_in, a, p, pol); });
}

// mu and its central gradient at lane k of the chunk, from the mu slab in
// global memory: mu(x), ((mu(x+1) - mu(x-1)) * 0.5) per axis (oracle op order).
template <int VVL>
struct MuGlobal {
    const FluidArgs &a;
    const Pos &p;
    __device__ __forceinline__ void operator()(int k, double &mu, double &gmx, double &gmy,
                                               double &gmz) const {
        const double *mc = a.mu + (long long)(p.z + 1) * a.PL;
        const int yp = wrapi(p.y + 1, a.ny), ym = wrapi(p.y - 1, a.ny);
        const int x = p.x0 + k;
        const long long r = (long long)p.y * a.nx;
        mu = __ldg(mc + r + x);
        gmx = Exact::mul(Exact::sub(__ldg(mc + r + wrapi(x + 1, a.nx)),
                                    __ldg(mc + r + wrapi(x - 1, a.nx))), 0.5);
        gmy = Exact::mul(Exact::sub(__ldg(mc + (long long)yp * a.nx + x),
                                    __ldg(mc + (long long)ym * a.nx + x)), 0.5);
        gmz = Exact::mul(Exact::sub(__ldg(mc + a.PL + r + x), __ldg(mc - a.PL + r + x)), 0.5);
    }
};

// physics 2: mu(x) and the stress-divergence force at lane k (oracle
// stress_force op order): F_a = -((D_x P_ax + D_y P_ay) + D_z P_az),
// D_b h = (h(+b) - h(-b)) * 0.5, P_aa = p_iso + ((kappa g_a) g_a),
// P_ab = (kappa g_a) g_b, from the aux arrays the mu kernel wrote.
template <int VVL>
struct StressGlobal {
    const FluidArgs &a;
    const Pos &p;
    __device__ __forceinline__ void operator()(int k, double &mu, double &Fx, double &Fy,
                                               double &Fz) const {
        using M = Exact;
        const long long PL = a.PL, as = a.astride;
        const long long c = (long long)(p.z + 1) * PL + (long long)p.y * a.nx + (p.x0 + k);
        const int x = p.x0 + k;
        // neighbour offsets from the centre: +-x (periodic), +-y (periodic), +-z (halo planes)
        const long long r = (long long)(p.z + 1) * PL + (long long)p.y * a.nx;
        const long long sp[3] = {r + wrapi(x + 1, a.nx),
                                 (long long)(p.z + 1) * PL + (long long)wrapi(p.y + 1, a.ny) * a.nx + x,
                                 c + PL};
        const long long sm[3] = {r + wrapi(x - 1, a.nx),
                                 (long long)(p.z + 1) * PL + (long long)wrapi(p.y - 1, a.ny) * a.nx + x,
                                 c - PL};
        mu = __ldg(a.mu + c);
        const double *piso = a.aux, *g[3] = {a.aux + as, a.aux + 2 * as, a.aux + 3 * as};
        double F[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            double dd[3];
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                double tp = M::mul(M::mul(a.kappa, __ldg(g[d] + sp[b])), __ldg(g[b] + sp[b]));
                double tm = M::mul(M::mul(a.kappa, __ldg(g[d] + sm[b])), __ldg(g[b] + sm[b]));
                if (d == b) {
                    tp = M::add(__ldg(piso + sp[b]), tp);
                    tm = M::add(__ldg(piso + sm[b]), tm);
                }
                dd[b] = M::mul(M::sub(tp, tm), 0.5);
            }
            F[d] = -M::add(M::add(dd[0], dd[1]), dd[2]);
        }
        Fx = F[0];
        Fy = F[1];
        Fz = F[2];
    }
};

template <int VVL, int MODE, int PHYS, int T1, int HINT, class MuFn>
__device__ __forceinline__ void cs_finish(const FluidArgs &a, const Pos &p, double (&F)[Q][VVL],
                                          double (&G)[Q][VVL], const MuFn &mufn) {
    using M = typename std::conditional<MODE == LTK_MODE_EXACT, Exact, Fast>::type;
    uint64_t pol_first = 0, pol_last = 0;
    if constexpr (HINT & 2) {
        pol_first = l2_evict_first();
        pol_last = l2_evict_last();
    }

    FSite st[VVL];
#pragma unroll
    for (int k = 0; k < VVL; ++k) st[k] = FSite{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0,
                                                0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    static_for<0, Q>([&](auto I) {
#pragma unroll
        for (int k = 0; k < VVL; ++k) faccum<I.value, M>(st[k], F[I.value][k]);
    });
    bool ok[VVL];
#pragma unroll
    for (int k = 0; k < VVL; ++k) {
#pragma unroll
        for (int i = 0; i < Q; ++i) st[k].phi = M::add(st[k].phi, G[i][k]);
        double gmx = 0.0, gmy = 0.0, gmz = 0.0;
        if constexpr (PHYS >= 1) mufn(k, st[k].mu, gmx, gmy, gmz);
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

    const long long off = (long long)p.y * a.SY + p.x0;       // row offset inside a plane
    const long long o = (long long)(p.z + 1) * a.SZ + off;
    static_for<0, Q>([&](auto I) {
        if constexpr (HINT & 2) {
            store_vec_pol<VVL>(a.f_out + I.value * a.SI + o, F[I.value], pol_first);
            store_vec_pol<VVL>(a.g_out + I.value * a.SI + o, G[I.value], pol_last);
        } else {
            store_vec<VVL>(a.f_out + I.value * a.SI + o, F[I.value]);
            store_vec<VVL>(a.g_out + I.value * a.SI + o, G[I.value]);
        }
        // halo images of the components that cross the z faces
        if constexpr (cz(I.value) < 0) {
            if (p.z == 0 && a.img_f_dn) {
                const long long h = (long long)(a.nzl + 1) * a.SZ + off;
                store_vec<VVL>(a.img_f_dn + I.value * a.SI + h, F[I.value]);
                store_vec<VVL>(a.img_g_dn + I.value * a.SI + h, G[I.value]);
            }
        }
        if constexpr (cz(I.value) > 0) {
            if (p.z == a.nzl - 1 && a.img_f_up) {
                store_vec<VVL>(a.img_f_up + I.value * a.SI + off, F[I.value]);
                store_vec<VVL>(a.img_g_up + I.value * a.SI + off, G[I.value]);
            }
        }
    });
    if ((p.z == 0 && a.img_f_dn) || (p.z == a.nzl - 1 && a.img_f_up))
        __threadfence_system();  // peer images visible before the progress signal
}

template <int VVL, int MODE, int PHYS, int T1, int HINT>
__device__ __forceinline__ void cs_site(const FluidArgs &a, const Pos &p) {
    double F[Q][VVL], G[Q][VVL];
    cs_load<VVL, HINT>(a, p, F, G);
    if constexpr (PHYS == 2) cs_finish<VVL, MODE, PHYS, T1, HINT>(a, p, F, G, StressGlobal<VVL>{a, p});
    else cs_finish<VVL, MODE, PHYS, T1, HINT>(a, p, F, G, MuGlobal<VVL>{a, p});
}

template <int VVL, int MODE, int PHYS, int T1, int HINT = 0>
__global__ void __launch_bounds__(128, VVL == 1 ? 4 : 1) k_collide_stream(const FluidArgs a) {
    Pos p;
    if (!thread_pos<VVL>(a, p)) return;
    cs_site<VVL, MODE, PHYS, T1, HINT>(a, p);
}

// ------------------------------------------------------------------ fused step
// k_cs_phi: collide-stream of planes [z_lo, z_lo + nplanes) AND phi of the
// NEXT state on planes [phi_lo, phi_hi), read back a few planes behind the
// collision front -- the k_phi pass over g' leaves the step.
// phi(x) = sum_i g'_i(x - c_i) reads g' on planes z-1..z+1, all written by
// this launch, so:
//  * work order: each CTA takes a ticket T (one atomicAdd); b = T mod ncta is
//    its work index, so every lower index of this launch is already resident
//    or finished; e = T div ncta counts this engine's launches (graph-replay
//    safe: counters are never reset, every launch takes exactly ncta tickets);
//  * warp w of CTA b handles collide threads [128 b + 32 w, +32) and the phi
//    threads lag_ctas*128 behind.  A warp first issues its collision loads,
//    then polls (ld.acquire) the completion counters of the planes its phi
//    sites pull from, then issues the phi loads (L2), then finishes the
//    collision and publishes its sites per plane (__syncwarp + one
//    red.release per plane).  No CTA barrier after the ticket: warps never
//    idle waiting for each other, so HBM requests stay in flight.
//  * lag_ctas covers > 3 planes + one CTA (host-checked), so the waited-on
//    planes belong to lower work indices: no deadlock; the host adds slack
//    planes so the poll is normally satisfied at once.
// Counters are 64-bit and cumulative: plane z is complete in launch e when
// done[z] >= (e + 1) * tpp.  phi arithmetic is phi_site's (index-order
// __dadd_rn): bitwise equal to k_phi.  phi planes never include 0 or nzl-1
// (no halo images from here; the engine forms those planes with k_phi).
__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_gpu_add(unsigned long long *p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int VVL, int MODE, int PHYS, int T1, int HINT>
__global__ void __launch_bounds__(128, VVL == 1 ? 4 : 1) k_cs_phi(const FluidArgs a) {
    __shared__ unsigned long long s_ticket;
    unsigned long long *const ticket = a.sync, *const done = a.sync + 1;
    if (threadIdx.x == 0) s_ticket = atomicAdd(ticket, 1ull);
    __syncthreads();
    const unsigned long long T = s_ticket;
    const unsigned b = (unsigned)(T % a.ncta);
    const unsigned long long target = (T / a.ncta + 1) * (unsigned long long)a.tpp;
    const long long tpp = a.tpp;
    const int lane = threadIdx.x & 31;
    const long long tw = (long long)b * 128 + (threadIdx.x & ~31);  // warp's first thread

    // ---- collision loads of this warp's sites
    const long long t = tw + lane;
    const bool has_cs = b < a.ncta_cs && t < a.nthreads;
    Pos pc;
    double F[Q][VVL], G[Q][VVL];
    if (has_cs) {
        pos_of<VVL>(a, (unsigned)t, a.z_lo, pc);
        cs_load<VVL, HINT>(a, pc, F, G);
    }
    // ---- phi of the next state, lag_ctas CTAs behind
    const long long nphi = (long long)(a.phi_hi - a.phi_lo) * tpp;
    const long long uw = tw - (long long)a.lag_ctas * 128;
    if (uw >= 0 && uw < nphi) {  // warp-uniform
        const long long u = uw + lane;
        const long long ul = (uw + 32 < nphi ? uw + 32 : nphi) - 1;
        const int zlo = a.phi_lo + (int)(uw / tpp) - 1, zhi = a.phi_lo + (int)(ul / tpp) + 1;
        if (lane <= zhi - zlo) {
            while (ld_acquire_gpu_u64(done + zlo + lane) < target) __nanosleep(64);
        }
        __syncwarp();
        if (u < nphi) {
            Pos p;
            pos_of<VVL>(a, (unsigned)u, a.phi_lo, p);
            phi_site<VVL, kLdCg, false>(a, p, a.g_out, a.phi_next, l2_evict_first());
        }
    }
    if (has_cs) cs_finish<VVL, MODE, PHYS, T1, HINT>(a, pc, F, G, MuGlobal<VVL>{a, pc});
    // ---- publish this warp's sites, one release per plane
    __syncwarp();
    if (b < a.ncta_cs && tw < a.nthreads) {
        const int z = has_cs ? (int)(t / tpp) : -1;
        const unsigned act = __ballot_sync(0xffffffffu, has_cs);
        const unsigned same = __match_any_sync(0xffffffffu, z);
        if (has_cs && lane == __ffs(same & act) - 1)
            red_release_gpu_add(done + a.z_lo + z, (unsigned long long)__popc(same & act));
    }
}

}  // namespace ltk
