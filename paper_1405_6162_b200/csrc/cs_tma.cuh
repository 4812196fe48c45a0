// cs_tma.cuh -- collide-stream with the pulled state staged in shared memory
// by the Tensor Memory Accelerator (warp-specialised, persistent).
//
// Why: k_collide_stream holds its 38 pulled values in registers (128 regs,
// 16 warps per SM), so the bytes in flight per SM are bounded by registers
// and the kernel sits right at the DRAM latency-bandwidth knee.  Here the
// loads are asynchronous bulk copies (cp.async.bulk, completing on an
// mbarrier): a ring of tiles per SM is in flight whatever the compute warps
// are doing.
//
// Tile = TX consecutive sites of one x-row (y, z).  Stage layout: 43 rows,
//   rows 0..18   f_i source row (y - cy_i, z - cz_i) of the pull
//   rows 19..37  g_i source row
//   rows 38..42  mu rows (y, z), (y+1, z), (y-1, z), (y, z+1), (y, z-1)
// FULL (TX == nx): a row is one bulk copy of nx doubles; the x-pull
// (c_x = +-1 reads x -+ 1) wraps inside the staged row.  Segments (TX < nx):
// rows carry a 2-double halo each side (16-byte aligned); components with
// c_x != 0 and the centre mu row are copied with their halo (pieces at the
// row edges wrap), the others copy the TX interior doubles only.
//
// Warp roles: warp 0 = producer (lane 0 arms the stage's full barrier with
// the byte count, lanes issue one row copy each); then NCW consumer warps
// taking 32-site chunks round-robin.  A consumer copies its sites' values
// from shared memory into registers, releases the chunk (empty barrier, one
// arrival per chunk) and then computes and stores, so the next tiles' copies
// are in flight during the math.
// Arithmetic: cs_finish (the code of k_collide_stream), mu from the staged
// rows in MuGlobal's op order -> bitwise identical results.
#pragma once

#include "stencil_tma.cuh"

namespace ltk {

constexpr int kTmaH = 2;             // x halo (doubles) each side, segment tiles
constexpr int kTmaRows = 2 * Q + 5;  // f, g, mu rows

template <int TX, bool FULL>
struct TmaGeom {
    static constexpr int H = FULL ? 0 : kTmaH;
    static constexpr int W = TX + 2 * H;  // staged row width (doubles)
    static constexpr size_t stage_bytes = (size_t)kTmaRows * W * 8;
    // bytes landing per tile: FULL -> every row TX; segments -> per
    // distribution 9 rows TX (c_x = 0) + 10 rows W, mu 1 row W + 4 rows TX
    static constexpr uint32_t tile_bytes =
        FULL ? (uint32_t)kTmaRows * TX * 8
             : (uint32_t)(2 * (9 * TX + 10 * W) + (W + 4 * TX)) * 8;
};

// D3Q19 velocity components for a runtime index (packed 2-bit tables: no
// local-memory arrays); same values as cx/cy/cz.
__device__ __forceinline__ int cx_rt(int i) {
    constexpr unsigned long long P = [] {
        unsigned long long v = 0;
        for (int k = 0; k < Q; ++k) v |= (unsigned long long)(cx(k) + 1) << (2 * k);
        return v;
    }();
    return (int)((P >> (2 * i)) & 3ull) - 1;
}
__device__ __forceinline__ int cy_rt(int i) {
    constexpr unsigned long long P = [] {
        unsigned long long v = 0;
        for (int k = 0; k < Q; ++k) v |= (unsigned long long)(cy(k) + 1) << (2 * k);
        return v;
    }();
    return (int)((P >> (2 * i)) & 3ull) - 1;
}
__device__ __forceinline__ int cz_rt(int i) {
    constexpr unsigned long long P = [] {
        unsigned long long v = 0;
        for (int k = 0; k < Q; ++k) v |= (unsigned long long)(cz(k) + 1) << (2 * k);
        return v;
    }();
    return (int)((P >> (2 * i)) & 3ull) - 1;
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Segment tile row: source elements [x0 - H, x0 + TX + H) of a periodic row
// into dst[0 .. W) (halo) or [x0, x0 + TX) into dst[H ..) (no halo).
template <int TX, bool FULL>
__device__ __forceinline__ void tma_tile_row(double *dst, const double *row, int x0, int nx,
                                             bool halo, uint64_t *bar) {
    using Gm = TmaGeom<TX, FULL>;
    if (FULL || !halo) {
        tma_row(dst + Gm::H, row + x0, TX * 8, bar);
        return;
    }
    const int left = x0 - Gm::H, right = x0 + TX + Gm::H;
    const int a0 = left > 0 ? left : 0, a1 = right < nx ? right : nx;
    tma_row(dst + (a0 - left), row + a0, (uint32_t)(a1 - a0) * 8, bar);
    if (left < 0) tma_row(dst, row + nx + left, (uint32_t)(-left) * 8, bar);
    if (right > nx) tma_row(dst + (nx - left), row, (uint32_t)(right - nx) * 8, bar);
}

struct TileXYZ {
    int x0, y, z;
};

template <int TX>
__device__ __forceinline__ TileXYZ tile_xyz(const FluidArgs &a, long long j) {
    const int nseg = a.nx / TX;
    TileXYZ t;
    t.x0 = (int)(j % nseg) * TX;
    const long long row = j / nseg;
    t.y = (int)(row % a.ny);
    t.z = a.z_lo + (int)(row / a.ny);
    return t;
}

// Producer lane `lane` issues its rows (lane, lane + 32) of tile t into `st`.
template <int TX, bool FULL>
__device__ __forceinline__ void cs_tma_issue(const FluidArgs &a, const TileXYZ &t, double *st,
                                             uint64_t *full, int lane) {
    using Gm = TmaGeom<TX, FULL>;
#pragma unroll 1
    for (int r = lane; r < kTmaRows; r += 32) {
        double *dst = st + (size_t)r * Gm::W;
        if (r < 2 * Q) {
            const int i = r < Q ? r : r - Q;
            const double *base = (r < Q ? a.f_in : a.g_in) + (long long)i * a.cstride;
            const long long zs = t.z + 1 - cz_rt(i);
            const int ys = wrapi(t.y - cy_rt(i), a.ny);
            tma_tile_row<TX, FULL>(dst, base + zs * a.PL + (long long)ys * a.nx, t.x0, a.nx,
                                   cx_rt(i) != 0, full);
        } else {
            const int m = r - 2 * Q;  // 0: (y,z) 1: y+1 2: y-1 3: z+1 4: z-1
            const int ys = m == 1 ? wrapi(t.y + 1, a.ny) : m == 2 ? wrapi(t.y - 1, a.ny) : t.y;
            const long long zs = t.z + 1 + (m == 3 ? 1 : m == 4 ? -1 : 0);
            tma_tile_row<TX, FULL>(dst, a.mu + zs * a.PL + (long long)ys * a.nx, t.x0, a.nx,
                                   m == 0, full);
        }
    }
}

// LDGSTS loader: producer thread `pt` of `npt` copies 16-byte units of tile t
// (cp.async.cg, L1 bypass) and then arrives on `full` when its copies have
// landed (cp.async.mbarrier.arrive.noinc).  Unit u of a staged row covers
// doubles [x0 - H + 2u, +2) of the periodic source row: the x wrap is a
// per-unit index wrap (nx even, so units never straddle the row end).
template <int TX, bool FULL>
__device__ __forceinline__ void cs_ldgsts_issue(const FluidArgs &a, const TileXYZ &t, double *st,
                                                uint64_t *full, int pt, int npt) {
    using Gm = TmaGeom<TX, FULL>;
    constexpr int UPR = Gm::W / 2;  // 16-byte units per staged row
    const int nx = a.nx;
#pragma unroll 1
    for (int r = 0; r < kTmaRows; ++r) {
        const double *row;
        if (r < 2 * Q) {
            const int i = r < Q ? r : r - Q;
            const double *base = (r < Q ? a.f_in : a.g_in) + (long long)i * a.cstride;
            const long long zs = t.z + 1 - cz_rt(i);
            row = base + zs * a.PL + (long long)wrapi(t.y - cy_rt(i), a.ny) * nx;
        } else {
            const int m = r - 2 * Q;
            const int ys = m == 1 ? wrapi(t.y + 1, a.ny) : m == 2 ? wrapi(t.y - 1, a.ny) : t.y;
            const long long zs = t.z + 1 + (m == 3 ? 1 : m == 4 ? -1 : 0);
            row = a.mu + zs * a.PL + (long long)ys * nx;
        }
        double *dst = st + (size_t)r * Gm::W;
        for (int u = pt; u < UPR; u += npt) {
            int xs = t.x0 - Gm::H + 2 * u;
            if (!FULL) xs = xs < 0 ? xs + nx : (xs >= nx ? xs - nx : xs);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + 2 * u)),
                         "l"(row + xs)
                         : "memory");
        }
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(full))
                 : "memory");
}

// grid: min(#tiles, #SMs); block: 32 * (1 + NCW); dynamic smem:
// STAGES * stage_bytes.  Tile j goes to CTA j mod grid; no inter-CTA
// dependencies.  Consumers are scheduled per 32-site chunk: consumer warp w
// takes chunks w, w + NCW, ... of the CTA's chunk sequence (TX/32 chunks per
// tile), so any number of consumer warps can share the ring; slot_tile keeps
// their barrier waits unambiguous.  Requires nx % TX == 0 (FULL: nx == TX) and
// VVL == 1.
template <int MODE, int PHYS, int T1, int TX, bool FULL, int STAGES, int NCW, int NPW>
__global__ void __launch_bounds__(32 * ((NPW > 0 ? NPW : 1) + NCW), 1) k_cs_tma(const FluidArgs a) {
    // NPW == 0: one TMA producer warp; NPW > 0: NPW LDGSTS producer warps
    using Gm = TmaGeom<TX, FULL>;
    constexpr int WPT = TX / 32;  // chunks per tile
    constexpr int PW = NPW > 0 ? NPW : 1;  // producer warps
    static_assert(NCW < STAGES * WPT, "consumer stride must stay below the ring depth");
    extern __shared__ __align__(128) double stage[];
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
    // slot_tile[s]: the CTA-local tile index k whose copies slot s is receiving
    // (written by the producer after the slot's previous tile was released).
    // mbarrier waits test a 1-bit phase parity against the current or the
    // immediately preceding phase only, and a consumer warp whose stride
    // exceeds one tile may reach slot s while the slot's previous fill is still
    // in flight -- the parity of its phase would alias the phase before that.
    // Waiting for the tag first pins the barrier to this tile's phase.
    __shared__ unsigned long long slot_tile[STAGES];  // accessed with shared-memory atomics
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], NPW > 0 ? 32 * NPW : 1);
            mbar_init(&empty[s], WPT);
            slot_tile[s] = ~0ull;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long ntiles = a.nthreads / TX;
    const long long G = gridDim.x;

    if (warp < PW) {  // ---------------- producer(s)
        long long k = 0;
        for (long long j = blockIdx.x; j < ntiles; j += G, ++k) {
            const int s = (int)(k % STAGES);
            if (k >= STAGES) {
                mbar_wait(&empty[s], (uint32_t)((k / STAGES - 1) & 1));
                // the consumers' generic-proxy reads of this slot happen before the
                // async-proxy (TMA / cp.async) writes that refill it
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            }
            if (threadIdx.x == 0)  // before the barrier is armed
                atomicExch(&slot_tile[s], (unsigned long long)k);
            __syncwarp();
            double *sb = stage + (size_t)s * (Gm::stage_bytes / 8);
            if constexpr (NPW == 0) {
                if (lane == 0) mbar_expect_tx(&full[s], Gm::tile_bytes);
                __syncwarp();
                cs_tma_issue<TX, FULL>(a, tile_xyz<TX>(a, j), sb, &full[s], lane);
            } else {
                cs_ldgsts_issue<TX, FULL>(a, tile_xyz<TX>(a, j), sb, &full[s], threadIdx.x,
                                          32 * NPW);
            }
        }
        return;
    }
    // ---------------- consumers
    const long long nmine = (ntiles - blockIdx.x + G - 1) / G;  // tiles of this CTA
    for (long long q = warp - PW;; q += NCW) {
        const long long k = q / WPT;
        if (k >= nmine) break;
        const int xl = (int)(q % WPT) * 32 + lane;
        const long long j = blockIdx.x + k * G;
        const int s = (int)(k % STAGES);
        while (atomicAdd(&slot_tile[s], 0ull) != (unsigned long long)k)  // slot receives tile k
            __nanosleep(32);
        mbar_wait(&full[s], (uint32_t)((k / STAGES) & 1));
        const double *sb = stage + (size_t)s * (Gm::stage_bytes / 8);
        double F[Q][1], G_[Q][1];
        static_for<0, Q>([&](auto I) {
            constexpr int C = cx(I.value);
            int xs = Gm::H + xl - C;
            if constexpr (FULL) xs = C > 0 ? (xl == 0 ? TX - 1 : xl - 1)
                                            : C < 0 ? (xl == TX - 1 ? 0 : xl + 1) : xl;
            F[I.value][0] = sb[(size_t)I.value * Gm::W + xs];
            G_[I.value][0] = sb[(size_t)(Q + I.value) * Gm::W + xs];
        });
        double mu_c = 0, gx = 0, gy = 0, gz = 0;
        if constexpr (PHYS == 1) {
            const double *mr = sb + (size_t)2 * Q * Gm::W;
            const int c = Gm::H + xl;
            const int cp = FULL ? (xl == TX - 1 ? 0 : xl + 1) : c + 1;
            const int cm = FULL ? (xl == 0 ? TX - 1 : xl - 1) : c - 1;
            mu_c = mr[c];
            gx = Exact::mul(Exact::sub(mr[cp], mr[cm]), 0.5);
            gy = Exact::mul(Exact::sub(mr[Gm::W + c], mr[2 * Gm::W + c]), 0.5);
            gz = Exact::mul(Exact::sub(mr[3 * Gm::W + c], mr[4 * Gm::W + c]), 0.5);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);  // chunk read: the values are in registers
        const TileXYZ t = tile_xyz<TX>(a, j);
        Pos p;
        p.x0 = t.x0 + xl;
        p.y = t.y;
        p.z = t.z;
        auto mufn = [&](int, double &m, double &gmx, double &gmy, double &gmz) {
            m = mu_c;
            gmx = gx;
            gmy = gy;
            gmz = gz;
        };
        cs_finish<1, MODE, PHYS, T1, 0>(a, p, F, G_, mufn);
    }
}

}  // namespace ltk

namespace ltk {
// cs_tma.cu
int num_sms();
bool cs_tma_ok(const FluidArgs &a, int vvl);
int launch_cs_tma(const FluidArgs &a, int mode, int phys, cudaStream_t st);
void preload_cs_tma(int nx);
}  // namespace ltk
