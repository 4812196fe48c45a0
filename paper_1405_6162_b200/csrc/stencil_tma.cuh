// stencil_tma.cuh -- chemical potential from a shared-memory staged phi tile,
// rows brought in by the Tensor Memory Accelerator (cp.async.bulk, 1-D bulk
// copies completing on an mbarrier).
//
// A CTA owns TY full x-rows and marches Z planes in z.  Its shared memory
// holds a ring of plane slots, each (TY + 2) rows x nx doubles (the rows
// y0-1 .. y0+TY, periodic in y): planes z-1, z, z+1 are read while the next
// planes are in flight.  Every phi value therefore crosses HBM/L2 about
// (TY+2)/TY * (Z+2)/Z times instead of once per stencil use, and the 7-point
// reads hit shared memory.  x is periodic inside a row (index wrap in smem).
// The arithmetic is mu_at's (fluid_kernels.cuh, oracle orc_mu op order), so
// the result is bitwise identical to k_mu.
#pragma once

#include "fluid_kernels.cuh"

namespace ltk {

// Measured on the B200 at 256^3 (k_mu time per step): TY 8 / 4 slots 0.096 ms,
// TY 4 / 6 slots 0.071 ms, TY 4 / 8 slots 0.084 ms, TY 2 / 8 slots 0.080 ms;
// the unstaged k_mu took 0.107 ms.
// Rows per CTA: 4 up to nx = 256, 2 beyond (keeps a CTA's ring <= ~75 KB so
// three CTAs share an SM).
constexpr int kMuZ = 16;     // planes per CTA
constexpr int kMuSlots = 6;  // plane ring: planes z-1..z+1 in use, 3 in flight

inline int mu_tma_rows(int nx) { return nx <= 256 ? 4 : 2; }

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 1-D TMA bulk copy global -> shared, completion counted on `bar`
__device__ __forceinline__ void tma_row(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Issue the TY+2 row copies of storage plane zs into ring slot `slot`.
template <int kMuTY>
__device__ __forceinline__ void load_plane(double *ring, uint64_t *bars, int slot, const FluidArgs &a,
                                           int y0, int zs) {
    const int nx = a.nx;
    double *dst = ring + (size_t)slot * (kMuTY + 2) * nx;
    const uint32_t row_bytes = (uint32_t)nx * 8u;
    mbar_expect_tx(&bars[slot], row_bytes * (kMuTY + 2));
    const double *plane = a.phi_in + (long long)zs * a.PL;
    for (int r = 0; r < kMuTY + 2; ++r) {
        const int y = wrapi(y0 - 1 + r, a.ny);
        tma_row(dst + (size_t)r * nx, plane + (long long)y * nx, row_bytes, &bars[slot]);
    }
}

// grid: (ny / kMuTY, ceil(nplanes / kMuZ)); block: up to 256 threads over x.
template <int kMuTY>
__global__ void __launch_bounds__(256) k_mu_tma(const FluidArgs a) {
    extern __shared__ __align__(128) double ring[];
    __shared__ __align__(8) uint64_t bars[kMuSlots];
    const int nx = a.nx;
    const int y0 = blockIdx.x * kMuTY;
    const int zb = a.z_lo + blockIdx.y * kMuZ;
    const int ze = min(zb + kMuZ, a.z_lo + a.nplanes);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kMuSlots; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // planes zb-1 .. ze (storage zs = z + 1) live in slot (z - zb + 1) % kMuSlots
    const int first = zb - 1, last = ze;
    if (threadIdx.x == 0)
        for (int z = first; z <= min(last, first + kMuSlots - 1); ++z)
            load_plane<kMuTY>(ring, bars, (z - first) % kMuSlots, a, y0, z + 1);
    const size_t slot_elems = (size_t)(kMuTY + 2) * nx;
    for (int z = zb; z < ze; ++z) {
        const int sm = (z - 1 - first) % kMuSlots, s0 = (z - first) % kMuSlots,
                  sp = (z + 1 - first) % kMuSlots;
        // k-th load of a slot completes phase k & 1
        mbar_wait(&bars[sm], ((z - 1 - first) / kMuSlots) & 1);
        mbar_wait(&bars[s0], ((z - first) / kMuSlots) & 1);
        mbar_wait(&bars[sp], ((z + 1 - first) / kMuSlots) & 1);
        const double *Pm = ring + sm * slot_elems, *P0 = ring + s0 * slot_elems,
                     *Pp = ring + sp * slot_elems;
        for (int r = 0; r < kMuTY; ++r) {
            const int y = y0 + r;
            const double *row = P0 + (size_t)(r + 1) * nx;
            for (int x = threadIdx.x; x < nx; x += blockDim.x) {
                const double ph = row[x];
                double s = row[x + 1 < nx ? x + 1 : 0];
                s = __dadd_rn(s, row[x > 0 ? x - 1 : nx - 1]);
                s = __dadd_rn(s, row[x + nx]);       // y + 1
                s = __dadd_rn(s, row[x - nx]);       // y - 1
                s = __dadd_rn(s, Pp[(size_t)(r + 1) * nx + x]);  // z + 1
                s = __dadd_rn(s, Pm[(size_t)(r + 1) * nx + x]);  // z - 1
                const double lap = __dsub_rn(s, __dmul_rn(6.0, ph));
                const double p3 = __dmul_rn(__dmul_rn(ph, ph), ph);
                const double mu = __dsub_rn(__dadd_rn(__dmul_rn(a.A, ph), __dmul_rn(a.B, p3)),
                                            __dmul_rn(a.kappa, lap));
                const long long off = (long long)y * nx + x;
                a.mu_out[(long long)(z + 1) * a.PL + off] = mu;
                if (z == 0 && a.img_mu_dn) {
                    a.img_mu_dn[(long long)(a.nzl + 1) * a.PL + off] = mu;
                    __threadfence_system();
                }
                if (z == a.nzl - 1 && a.img_mu_up) {
                    a.img_mu_up[off] = mu;
                    __threadfence_system();
                }
            }
        }
        __syncthreads();  // every thread is done with plane z-1's slot
        const int nz_next = z - 1 + kMuSlots;  // plane that reuses slot sm
        if (threadIdx.x == 0 && nz_next <= last) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            load_plane<kMuTY>(ring, bars, sm, a, y0, nz_next + 1);
        }
    }
}

// ------------------------------------------------------------------ k_mu_col
// Register 2.5-D stencil: a (32 x 8) block of (x, y) columns marches kMuColZ
// planes in z, phi(z-1), phi(z), phi(z+1) rolling in registers; x +- 1 by
// warp shuffle (lanes 0/31 load across the warp edge, periodic), y +- 1 from
// L1/L2 (rows shared with the neighbouring warps of the block).  Per plane a
// thread issues one new-plane load plus two row loads, all independent of the
// arithmetic, so the kernel streams phi at DRAM speed instead of the
// per-SM bulk-copy rate that bounds k_mu_tma.  Op order is mu_at's: bitwise
// identical to k_mu / k_mu_tma.  Requires nx % 32 == 0, ny % 8 == 0.
constexpr int kMuColZ = 16;

// (Measured at 256^3: 0.079-0.085 ms per launch; a register ring prefetching
// 1-4 planes ahead and 8-32 planes per block changed nothing.)
// mu of one site from its 7-point phi neighbourhood (reference op order), stored
// with the stress outputs and the halo images where they apply.
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
    const long long PL = a.PL;
    a.mu_out[(long long)(z + 1) * PL + off] = mu;
    if (a.aux) stress_store(a, z, off, pc, mu, vxp, vxm, vyp, vym, pp, pm);
    bool img = false;
    if (z == 0 && a.img_mu_dn) {
        a.img_mu_dn[(long long)(a.nzl + 1) * PL + off] = mu;
        img = true;
    }
    if (z == a.nzl - 1 && a.img_mu_up) {
        a.img_mu_up[off] = mu;
        img = true;
    }
    if (img) __threadfence_system();
}

template <int ZC = kMuColZ>
__global__ void __launch_bounds__(256) k_mu_col(const FluidArgs a) {
    const int lane = threadIdx.x, nx = a.nx;
    const int x = blockIdx.x * 32 + lane, y = blockIdx.y * 8 + threadIdx.y;
    const int zb = a.z_lo + blockIdx.z * ZC;
    const int ze = min(zb + ZC, a.z_lo + a.nplanes);
    const long long PL = a.PL;
    const int yp = wrapi(y + 1, a.ny), ym = wrapi(y - 1, a.ny);
    const int xe = lane == 0 ? wrapi(x - 1, nx) : wrapi(x + 1, nx);  // across the warp edge
    const double *ph = a.phi_in;
    const long long r0 = (long long)y * nx, rp = (long long)yp * nx, rm = (long long)ym * nx;
    double pm = __ldg(ph + (long long)zb * PL + r0 + x);        // storage zs = z + 1
    double pc = __ldg(ph + (long long)(zb + 1) * PL + r0 + x);
#pragma unroll 2
    for (int z = zb; z < ze; ++z) {
        const double *c = ph + (long long)(z + 1) * PL;
        const double pp = __ldg(c + PL + r0 + x);
        const double vyp = __ldg(c + rp + x), vym = __ldg(c + rm + x);
        const double edge = (lane == 0 || lane == 31) ? __ldg(c + r0 + xe) : 0.0;
        double vxp = __shfl_down_sync(0xffffffffu, pc, 1);
        double vxm = __shfl_up_sync(0xffffffffu, pc, 1);
        if (lane == 31) vxp = edge;
        if (lane == 0) vxm = edge;
        mu_site_store(a, z, r0 + x, pm, pc, pp, vxp, vxm, vyp, vym);
        pm = pc;
        pc = pp;
    }
}

// The same stencil with the block's ZC + 2 centre planes loaded before any
// arithmetic: that many HBM loads in flight per thread (k_mu_col has about
// one), the memory-level parallelism a 16 B/site kernel lacks at 32 warps/SM.
// The y and warp-edge neighbours are then L1 hits (the rows of the block's
// other warps) and are loaded as they are used.  Measured (256^3, B200):
// 0.092 ms vs k_mu_col's 0.099; ZC = 16 (80 regs), prefetching the next
// plane's neighbours (70 regs) or batching the block's outer y rows (78 regs)
// all lose occupancy and run 0.097-0.12 ms.
template <int ZC, int MINB = 5>  // 5 blocks/SM: 48 regs (0.091 ms; 4: 62 regs 0.094, 6: spills 0.105)
__global__ void __launch_bounds__(256, MINB) k_mu_blk(const FluidArgs a) {
    const int lane = threadIdx.x, nx = a.nx;
    const int x = blockIdx.x * 32 + lane, y = blockIdx.y * 8 + threadIdx.y;
    const int zb = a.z_lo + blockIdx.z * ZC;
    const int n = min(ZC, a.z_lo + a.nplanes - zb);
    const long long PL = a.PL;
    const int yp = wrapi(y + 1, a.ny), ym = wrapi(y - 1, a.ny);
    const int xe = lane == 0 ? wrapi(x - 1, nx) : wrapi(x + 1, nx);
    const bool edge_lane = lane == 0 || lane == 31;
    const double *ph = a.phi_in + (long long)zb * PL + x;  // storage plane zb (= z - 1 of the first)
    const long long r0 = (long long)y * nx, rp = (long long)yp * nx, rm = (long long)ym * nx;
    double C[ZC + 2];
#pragma unroll
    for (int k = 0; k < ZC + 2; ++k) C[k] = k < n + 2 ? __ldg(ph + k * PL + r0) : 0.0;
#pragma unroll
    for (int k = 0; k < ZC; ++k) {
        if (k < n) {  // n is uniform over the block: the shuffles see full warps
            const double *c = ph + (k + 1) * PL;
            const double vyp = __ldg(c + rp), vym = __ldg(c + rm);
            const double edge = edge_lane ? __ldg(c + r0 + (xe - x)) : 0.0;
            double vxp = __shfl_down_sync(0xffffffffu, C[k + 1], 1);
            double vxm = __shfl_up_sync(0xffffffffu, C[k + 1], 1);
            if (lane == 31) vxp = edge;
            if (lane == 0) vxm = edge;
            mu_site_store(a, zb + k, r0 + x, C[k], C[k + 1], C[k + 2], vxp, vxm, vyp, vym);
        }
    }
}
constexpr int kMuBlkZ = 8;

// The same stencil with the block's phi tile -- ZC + 2 planes x (8 + 2) rows x
// (32 + 2) columns, halos included -- copied into shared memory by per-thread
// cp.async (LDGSTS): the loads in flight hold no registers.  48 registers and
// 27 KB of shared memory give 5 blocks per SM.  mu op order unchanged
// (mu_site_store).  Measured (256^3, B200): 0.070 ms vs k_mu_blk's 0.091.
// 16 planes (64 regs, 49 KB) run 0.075 ms.  Capping at 40 regs (6 blocks)
// changes nothing; 32 regs (8 blocks) spills and runs 0.091 ms.
template <int ZC>
__global__ void __launch_bounds__(256) k_mu_lds(const FluidArgs a) {
    __shared__ double t[ZC + 2][10][34];
    const int lane = threadIdx.x, wy = threadIdx.y, nx = a.nx;
    const int x = blockIdx.x * 32 + lane, y = blockIdx.y * 8 + wy;
    const int zb = a.z_lo + blockIdx.z * ZC;
    const int n = min(ZC, a.z_lo + a.nplanes - zb);
    const long long PL = a.PL;
    const double *ph = a.phi_in + (long long)zb * PL;  // storage plane zb (= z - 1 of the first)
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

constexpr int kMuLdsZ = 8;

inline bool mu_col_ok(const FluidArgs &a) { return a.nx % 32 == 0 && a.ny % 8 == 0; }

inline size_t mu_tma_smem(const FluidArgs &a) {
    return (size_t)kMuSlots * (mu_tma_rows(a.nx) + 2) * a.nx * 8;
}

inline bool mu_tma_ok(const FluidArgs &a) {
    return !a.aux && a.ny % mu_tma_rows(a.nx) == 0 && a.nx % 2 == 0 &&
           mu_tma_smem(a) <= 200 * 1024;  // (no stress outputs)
}

}  // namespace ltk
