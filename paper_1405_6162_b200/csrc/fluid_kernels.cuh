// fluid_kernels.cuh -- device kernels of the full D3Q19 binary-fluid timestep
// (builder-defined extension).
//
// Slab layout: x fastest, z slowest.  f/g element (component
// i, storage plane zs, row y, x) at i*SI + zs*SZ + y*SY + x, storage plane
// zs = z + 1 (halo planes zs = 0 and nzl + 1); SoA (SI, SZ, SY) =
// (cstride, nx*ny, nx) or row-blocked (nx, ny*19*nx, 19*nx).  phi planes are
// plane-major with one halo plane per side (zs = z + 1, nzl + 2 planes); mu
// (and the stress form's aux arrays) with two (zs = z + 2, nzl + 4 planes),
// because the filtered potential force reads mu at z +- 2.
//
// One timestep = k_phi -> k_mu -> k_collide_stream (pull scheme):
//   k_phi   phi(x) = sum_i g_i(x - c_i)                        [g pulled]
//   k_mu    mu = A phi + B phi^3 - kappa lap7(phi)              [phi stencil]
//   k_cs    pull f, g; force from the phi / mu stencils; Guo-forced BGK for
//           f, chemical-potential g_eq; aligned store.
// Halo images: a kernel that produces an owned plane some other plane's
// stencil needs across a slab face also stores it straight into the halo
// plane that needs it -- into this slab's own halos on one GPU (periodic z,
// no halo kernels), into the neighbours' buffers mapped with CUDA IPC with
// the peer transport (the halo exchange fused into the producing kernels as
// NVLink stores), nowhere with NCCL (the engine exchanges faces).
#pragma once

#include "ltk_common.cuh"

namespace ltk {

struct FluidArgs {
    const double *f_in, *g_in;  // state read (post-collision of the last step)
    double *f_out, *g_out;      // state written
    const double *phi;          // phi slab read by k_mu / k_collide_stream
    double *phi_out;            // phi slab written by k_phi
    const double *mu;           // mu slab read by k_collide_stream
    double *mu_out;             // mu slab written by k_mu
    // physics 2 (stress form): p_iso, d_x phi, d_y phi, d_z phi in mu's layout
    // at aux + k * astride (after mu in mu's allocation); written by k_mu
    double *aux;
    long long astride;
    long long *err;  // the engine's / stream's error word (flag_singular)
    int nx, ny, nzl, z_lo, nplanes;
    int wrap_local;  // images into this slab's own halos (periodic z, one slab)
    // halo image targets (nullptr = none): buffers of the slab above (up) /
    // below (dn); f/g point at the state being written; aux images follow mu's
    double *img_f_up, *img_g_up, *img_f_dn, *img_g_dn;
    double *img_phi_up, *img_phi_dn, *img_mu_up, *img_mu_dn;
    long long PL;
    long long SI, SZ, SY;
    long long nthreads;       // threads of this launch
    long long nz_global, z0;  // for error-site reporting in host order
    double wv[Q];
    double lam[Q];
    double sw[Q];  // srcpre * wv[i] (host, the same RN product the oracle forms per site)
    double cs2, tau_f, tau_g, A, B, kappa, gamma;
    // derived (host-computed once, each the same IEEE expression as the oracle)
    double c1, c2, cs2sq, srcpre;                                 // 2cs2, (2cs2)cs2, cs2*cs2, 1 - 0.5/tau_f
    double inv_tau_f, inv_tau_g, a1, a2, a3, inv_cs2, inv_cs2sq;  // reciprocals
};

// thread -> (x0, y, z) of a VVL-site row segment
struct Pos {
    int x0, y, z;
};

template <int VVL>
__device__ __forceinline__ bool thread_pos(const FluidArgs &a, Pos &p) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.nthreads) return false;
    const unsigned tt = (unsigned)t;
    const unsigned nxv = (unsigned)(a.nx / VVL);
    const unsigned row = tt / nxv;
    p.x0 = (int)(tt - row * nxv) * VVL;
    p.y = (int)(row % (unsigned)a.ny);
    p.z = a.z_lo + (int)(row / (unsigned)a.ny);
    return true;
}

__device__ __forceinline__ int wrapi(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }
// |v| < 2n (offsets of +-2 on extents >= 1)
__device__ __forceinline__ int wrap2(int v, int n) { return wrapi(wrapi(v, n), n); }

// Pull the VVL values of component I at sites (x0..x0+VVL-1, y, zs) from
// (x - cx, y - cy, zs - cz).  cx == 0 -> one aligned vector load.
template <int I, int VVL>
__device__ __forceinline__ void pull(double (&v)[VVL], const double *base, const FluidArgs &a,
                                     const Pos &p) {
    const int ys = wrapi(p.y - cy(I), a.ny);
    const double *row = base + (long long)I * a.SI + (long long)(p.z + 1 - cz(I)) * a.SZ +
                        (long long)ys * a.SY;
    if constexpr (cx(I) == 0) {
        load_vec<VVL>(v, row + p.x0);
    } else {
#pragma unroll
        for (int k = 0; k < VVL; ++k) v[k] = __ldg(row + wrapi(p.x0 + k - cx(I), a.nx));
    }
}

// ------------------------------------------------------------------ phi
template <int VVL>
__global__ void __launch_bounds__(128) k_phi(const FluidArgs a) {
    Pos p;
    if (!thread_pos<VVL>(a, p)) return;
    double phi[VVL];
#pragma unroll
    for (int k = 0; k < VVL; ++k) phi[k] = 0.0;
    double v[Q][VVL];  // all loads issued before the first add
    static_for<0, Q>([&](auto I) { pull<I.value, VVL>(v[I.value], a.g_in, a, p); });
    static_for<0, Q>([&](auto I) {
#pragma unroll
        for (int k = 0; k < VVL; ++k) phi[k] = __dadd_rn(phi[k], v[I.value][k]);
    });
    const long long off = (long long)p.y * a.nx + p.x0;
    store_vec<VVL>(a.phi_out + (long long)(p.z + 1) * a.PL + off, phi);
    // halo images for the stencils of the neighbouring slabs (or this one)
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
// mu-layout halo planes an owned plane z feeds: the slab above reads our
// planes nzl-2, nzl-1 as its z = -2, -1 (storage 0, 1); the slab below reads
// our planes 0, 1 as its z = nzl, nzl+1 (storage nzl+2, nzl+3).  One slab
// (wrap_local): halo plane hz holds plane hz mod nzl, which also covers nzl = 1.
__device__ __forceinline__ int modi(int v, int n) { return ((v % n) + n) % n; }

template <class Store>
__device__ __forceinline__ bool mu_images(const FluidArgs &a, int z, Store store) {
    // only planes 0, 1, nzl-2, nzl-1 feed halo planes (any nzl): skip the
    // source-plane arithmetic (two integer modulos per image) everywhere else
    if (z >= 2 && z < a.nzl - 2) return false;
    bool img = false;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int hz_up = k - 2;       // the slab above's halo plane
        const int hz_dn = a.nzl + k;   // the slab below's halo plane
        const int src_up = a.wrap_local ? modi(hz_up, a.nzl) : a.nzl + hz_up;
        const int src_dn = a.wrap_local ? modi(hz_dn, a.nzl) : k;
        if (a.img_mu_up && z == src_up) {
            store(a.img_mu_up, (long long)(hz_up + 2) * a.PL);
            img = true;
        }
        if (a.img_mu_dn && z == src_dn) {
            store(a.img_mu_dn, (long long)(hz_dn + 2) * a.PL);
            img = true;
        }
    }
    return img;
}

// physics 2 side outputs of the mu kernels: p_iso and the central gradient of
// phi (oracle orc_stress op order).
__device__ __forceinline__ void stress_values(const FluidArgs &a, double ph, double mu, double xp,
                                              double xm, double yp, double ym, double zp,
                                              double zm, double (&v)[4]) {
    using M = Exact;
    const double gx = M::mul(M::sub(xp, xm), 0.5);
    const double gy = M::mul(M::sub(yp, ym), 0.5);
    const double gz = M::mul(M::sub(zp, zm), 0.5);
    const double gsq = M::add(M::add(M::mul(gx, gx), M::mul(gy, gy)), M::mul(gz, gz));
    const double pp = M::mul(ph, ph);
    const double fb = M::add(M::mul(M::mul(0.5, a.A), pp), M::mul(M::mul(0.25, a.B), M::mul(pp, pp)));
    v[0] = M::sub(M::sub(M::mul(ph, mu), fb), M::mul(M::mul(0.5, a.kappa), gsq));
    v[1] = gx;
    v[2] = gy;
    v[3] = gz;
}

// mu of one site from its 7-point phi neighbourhood, stored with the stress
// outputs and the halo images where they apply (oracle orc_mu op order):
// mu = (A phi + B phi^3) - kappa lap, lap = (((((phi(x+1) + phi(x-1)) + phi(y+1))
//      + phi(y-1)) + phi(z+1)) + phi(z-1)) - 6 phi.
__device__ __forceinline__ void mu_site_store(const FluidArgs &a, int z, long long off, double pm,
                                              double pc, double pp, double vxp, double vxm,
                                              double vyp, double vym) {
    double s = __dadd_rn(vxp, vxm);
    s = __dadd_rn(s, vyp);
    s = __dadd_rn(s, vym);
    s = __dadd_rn(s, pp);
    s = __dadd_rn(s, pm);
    const double lap = __dsub_rn(s, __dmul_rn(6.0, pc));
    const double p3 = __dmul_rn(__dmul_rn(pc, pc), pc);
    const double mu = __dsub_rn(__dadd_rn(__dmul_rn(a.A, pc), __dmul_rn(a.B, p3)),
                                __dmul_rn(a.kappa, lap));
    const long long o = (long long)(z + 2) * a.PL + off;
    a.mu_out[o] = mu;
    double sv[4];
    if (a.aux) {
        stress_values(a, pc, mu, vxp, vxm, vyp, vym, pp, pm, sv);
#pragma unroll
        for (int k = 0; k < 4; ++k) a.aux[k * a.astride + o] = sv[k];
    }
    const bool img = mu_images(a, z, [&](double *dst, long long plane) {
        dst[plane + off] = mu;
        if (a.aux)
#pragma unroll
            for (int k = 0; k < 4; ++k) dst[(k + 1) * a.astride + plane + off] = sv[k];
    });
    if (img) __threadfence_system();
}

// Plain stencil: one thread per VVL sites, neighbours from L1/L2 (any shape).
template <int VVL>
__global__ void __launch_bounds__(128) k_mu(const FluidArgs a) {
    Pos p;
    if (!thread_pos<VVL>(a, p)) return;
    const double *c = a.phi + (long long)(p.z + 1) * a.PL;
    const long long r0 = (long long)p.y * a.nx;
    const long long rp = (long long)wrapi(p.y + 1, a.ny) * a.nx, rm = (long long)wrapi(p.y - 1, a.ny) * a.nx;
#pragma unroll
    for (int k = 0; k < VVL; ++k) {
        const int x = p.x0 + k;
        mu_site_store(a, p.z, r0 + x, __ldg(c - a.PL + r0 + x), __ldg(c + r0 + x),
                      __ldg(c + a.PL + r0 + x), __ldg(c + r0 + wrapi(x + 1, a.nx)),
                      __ldg(c + r0 + wrapi(x - 1, a.nx)), __ldg(c + rp + x), __ldg(c + rm + x));
    }
}

// Tile stencil (default where nx % 32 == 0 and ny % 8 == 0): a (32 x 8)
// column block copies its phi tile -- ZC + 2 planes x 10 rows x 34 columns,
// halos included -- into shared memory with per-thread cp.async (LDGSTS), so
// the loads in flight hold no registers, then every neighbour is a
// shared-memory read.  48 registers, 27 KB: 5 blocks per SM.  Measured
// (round 1, 256^3): 0.070 ms vs 0.091-0.107 ms for register-resident forms.
constexpr int kMuTileZ = 8;

inline bool mu_tile_ok(int nx, int ny) { return nx % 32 == 0 && ny % 8 == 0; }

template <int ZC>
__global__ void __launch_bounds__(256) k_mu_tile(const FluidArgs a) {
    __shared__ double t[ZC + 2][10][34];
    const int lane = threadIdx.x, wy = threadIdx.y, nx = a.nx;
    const int x = blockIdx.x * 32 + lane, y = blockIdx.y * 8 + wy;
    const int zb = a.z_lo + blockIdx.z * ZC;
    const int n = min(ZC, a.z_lo + a.nplanes - zb);
    const long long PL = a.PL;
    const double *ph = a.phi + (long long)zb * PL;  // storage plane zb = z - 1 of the first
    const long long r0 = (long long)y * nx;
    auto cp8 = [](double *dst, const double *src) {
        const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(src) : "memory");
    };
#pragma unroll
    for (int k = 0; k < ZC + 2; ++k)
        if (k < n + 2) cp8(&t[k][wy + 1][lane + 1], ph + k * PL + r0 + x);
    // y halo rows (outer warps) and x halo columns (edge lanes) of the computed planes
    if (wy == 0 || wy == 7) {
        const long long rh = (long long)wrapi(wy == 0 ? y - 1 : y + 1, a.ny) * nx;
        const int row = wy == 0 ? 0 : 9;
#pragma unroll
        for (int k = 1; k < ZC + 1; ++k)
            if (k < n + 1) cp8(&t[k][row][lane + 1], ph + k * PL + rh + x);
    }
    if (lane == 0 || lane == 31) {
        const int xh = wrapi(lane == 0 ? x - 1 : x + 1, nx);
        const int col = lane == 0 ? 0 : 33;
#pragma unroll
        for (int k = 1; k < ZC + 1; ++k)
            if (k < n + 1) cp8(&t[k][wy + 1][col], ph + k * PL + r0 + xh);
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int k = 0; k < ZC; ++k) {
        if (k < n) {
            const int r = wy + 1, c = lane + 1;
            mu_site_store(a, zb + k, r0 + x, t[k][r][c], t[k + 1][r][c], t[k + 2][r][c],
                          t[k + 1][r][c + 1], t[k + 1][r][c - 1], t[k + 1][r + 1][c],
                          t[k + 1][r - 1][c]);
        }
    }
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

// Filtered potential force along one axis (oracle orc_potential_force):
//   h(x) = -(phi(x) * ((mu(x+1) - mu(x-1)) * 0.5)),
//   F = ((h(x-1) + h(x+1)) + (h(x) + h(x))) * 0.25,
// from phi at x, x+-1 and mu at x, x+-1, x+-2 along the axis.
__device__ __forceinline__ double force_axis(double ph0, double php, double phm, double mu0,
                                             double mp1, double mm1, double mp2, double mm2) {
    using M = Exact;
    const double h0 = -M::mul(ph0, M::mul(M::sub(mp1, mm1), 0.5));
    const double hp = -M::mul(php, M::mul(M::sub(mp2, mu0), 0.5));
    const double hm = -M::mul(phm, M::mul(M::sub(mu0, mm2), 0.5));
    return M::mul(M::add(M::add(hm, hp), M::add(h0, h0)), 0.25);
}

// physics 1: mu(x) and the filtered potential force at lane k of the chunk,
// from the phi and mu slabs.  phi(x) from the slab equals the in-register sum
// of the pulled g bitwise (k_phi forms it from the same state in index order).
template <int VVL>
struct ForcePot {
    const FluidArgs &a;
    const Pos &p;
    __device__ __forceinline__ void operator()(int k, double &mu, double &Fx, double &Fy,
                                               double &Fz) const {
        const int x = p.x0 + k, nx = a.nx, ny = a.ny;
        const long long PL = a.PL;
        const double *pc = a.phi + (long long)(p.z + 1) * PL + (long long)p.y * nx;
        const double *mc = a.mu + (long long)(p.z + 2) * PL + (long long)p.y * nx;
        const int xp1 = wrapi(x + 1, nx), xm1 = wrapi(x - 1, nx);
        const int xp2 = wrap2(x + 2, nx), xm2 = wrap2(x - 2, nx);
        const long long yp1 = (long long)(wrapi(p.y + 1, ny) - p.y) * nx,
                        ym1 = (long long)(wrapi(p.y - 1, ny) - p.y) * nx,
                        yp2 = (long long)(wrap2(p.y + 2, ny) - p.y) * nx,
                        ym2 = (long long)(wrap2(p.y - 2, ny) - p.y) * nx;
        const double ph0 = __ldg(pc + x);
        mu = __ldg(mc + x);
        Fx = force_axis(ph0, __ldg(pc + xp1), __ldg(pc + xm1), mu, __ldg(mc + xp1),
                        __ldg(mc + xm1), __ldg(mc + xp2), __ldg(mc + xm2));
        Fy = force_axis(ph0, __ldg(pc + yp1 + x), __ldg(pc + ym1 + x), mu, __ldg(mc + yp1 + x),
                        __ldg(mc + ym1 + x), __ldg(mc + yp2 + x), __ldg(mc + ym2 + x));
        Fz = force_axis(ph0, __ldg(pc + PL + x), __ldg(pc - PL + x), mu, __ldg(mc + PL + x),
                        __ldg(mc - PL + x), __ldg(mc + 2 * PL + x), __ldg(mc - 2 * PL + x));
    }
};

// physics 2: mu(x) and the stress-divergence force at lane k (oracle
// stress_force op order): F_a = -((D_x P_ax + D_y P_ay) + D_z P_az),
// D_b h = (h(+b) - h(-b)) * 0.5, P_aa = p_iso + ((kappa g_a) g_a),
// P_ab = (kappa g_a) g_b, from the aux arrays the mu kernel wrote.
template <int VVL>
struct ForceStress {
    const FluidArgs &a;
    const Pos &p;
    __device__ __forceinline__ void operator()(int k, double &mu, double &Fx, double &Fy,
                                               double &Fz) const {
        using M = Exact;
        const long long PL = a.PL, as = a.astride;
        const int x = p.x0 + k;
        const long long r = (long long)(p.z + 2) * PL + (long long)p.y * a.nx;
        const long long c = r + x;
        const long long sp[3] = {r + wrapi(x + 1, a.nx),
                                 (long long)(p.z + 2) * PL + (long long)wrapi(p.y + 1, a.ny) * a.nx + x,
                                 c + PL};
        const long long sm[3] = {r + wrapi(x - 1, a.nx),
                                 (long long)(p.z + 2) * PL + (long long)wrapi(p.y - 1, a.ny) * a.nx + x,
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

// Site-wide quantities after the moments (oracle collide_site op order).
template <int MODE, int PHYS>
__device__ __forceinline__ void fsite_finish(FSite &s, const FluidArgs &a) {
    using M = Exact;
    if constexpr (MODE == LTK_MODE_EXACT) {
        const double rr = __drcp_rn(s.rho);  // RN(1/rho): three divisions by rho
        if constexpr (PHYS >= 1) {
            s.ux = div_rcp(M::add(s.jx, M::mul(0.5, s.Fx)), s.rho, rr);
            s.uy = div_rcp(M::add(s.jy, M::mul(0.5, s.Fy)), s.rho, rr);
            s.uz = div_rcp(M::add(s.jz, M::mul(0.5, s.Fz)), s.rho, rr);
            s.uF = M::add(M::add(M::mul(s.ux, s.Fx), M::mul(s.uy, s.Fy)), M::mul(s.uz, s.Fz));
            s.psi = M::sub(M::mul(a.gamma, s.mu), M::mul(s.phi, a.cs2));
        } else {
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

// One VVL-site chunk: pull f, g (38 values per site held in registers, one
// HBM read + one write each), force and mu from the stencils, collide, store
// aligned, plus the halo images of the components that cross a z face.
template <int VVL, int MODE, int PHYS, int T1>
__device__ __forceinline__ void cs_site(const FluidArgs &a, const Pos &p) {
    using M = typename std::conditional<MODE == LTK_MODE_EXACT, Exact, Fast>::type;
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
#pragma unroll
    for (int k = 0; k < VVL; ++k) {
#pragma unroll
        for (int i = 0; i < Q; ++i) st[k].phi = M::add(st[k].phi, G[i][k]);
        if constexpr (PHYS == 1) ForcePot<VVL>{a, p}(k, st[k].mu, st[k].Fx, st[k].Fy, st[k].Fz);
        if constexpr (PHYS == 2) ForceStress<VVL>{a, p}(k, st[k].mu, st[k].Fx, st[k].Fy, st[k].Fz);
        ok[k] = !(st[k].rho <= 0.0);
        if (ok[k]) {
            fsite_finish<MODE, PHYS>(st[k], a);
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

    const long long off = (long long)p.y * a.SY + p.x0;  // row offset inside a plane
    const long long o = (long long)(p.z + 1) * a.SZ + off;
    static_for<0, Q>([&](auto I) {
        store_vec<VVL>(a.f_out + I.value * a.SI + o, F[I.value]);
        store_vec<VVL>(a.g_out + I.value * a.SI + o, G[I.value]);
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

template <int VVL, int MODE, int PHYS, int T1>
__global__ void __launch_bounds__(128, VVL == 1 ? 4 : 1) k_collide_stream(const FluidArgs a) {
    Pos p;
    if (!thread_pos<VVL>(a, p)) return;
    cs_site<VVL, MODE, PHYS, T1>(a, p);
}

}  // namespace ltk
