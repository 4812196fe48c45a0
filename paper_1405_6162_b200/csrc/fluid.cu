// fluid.cu -- the full D3Q19 binary-fluid timestep on B200: C-ABI launchers
// of the kernels in fluid_kernels.cuh, host-order <-> slab transposes, halo
// faces, and the C++ step engine (single GPU periodic, or z-slabs with NCCL
// halo exchange overlapped with the interior planes).
//
// No reference counterpart (reference pkg/README.md:34-35: collision only);
// specification in DESIGN.md §2-§5.  The collision arithmetic is the
// reference's (kernels.py:89-125) with the free-energy force terms added.
#include <cuda.h>  // CUresult / CUdeviceptr for the driver entry point (no libcuda link)
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl.so.2 is dlopen'ed at run time

#include <algorithm>
#include <cstring>
#include <initializer_list>
#include <new>
#include <vector>

#include "cs_tma.cuh"

namespace ltk {

// ------------------------------------------------------------------ helpers

static int check_slab(const ltk_slab *s, int vvl) {
    if (!s || s->nx < 1 || s->ny < 1 || s->nzl < 1)
        return fail(LTK_ERR_SHAPE, "invalid slab extents");
    if (s->cstride < (s->nzl + 2) * s->nx * s->ny)
        return fail(LTK_ERR_SHAPE, "cstride %lld < (nzl+2)*nx*ny", (long long)s->cstride);
    if (vvl != 1 && vvl != 2 && vvl != 4)
        return fail(LTK_ERR_PLAN, "fluid kernels support vvl 1, 2, 4 (got %d)", vvl);
    if (s->nx % vvl) return fail(LTK_ERR_PLAN, "vvl %d does not divide nx %lld", vvl,
                                 (long long)s->nx);
    if ((s->nx * s->ny) % 2 || s->cstride % 2)
        return fail(LTK_ERR_SHAPE, "nx*ny and cstride must be even (16-byte vector rows)");
    if ((long long)s->nx * s->ny * (s->nzl + 2) >= (1LL << 31))
        return fail(LTK_ERR_SHAPE, "slab too large for 32-bit thread indexing");
    return LTK_OK;
}

static void fill_args(FluidArgs &a, const ltk_slab *s, const ltk_fluid_params *p) {
    memset(&a, 0, sizeof a);
    a.nx = (int)s->nx;
    a.ny = (int)s->ny;
    a.nzl = (int)s->nzl;
    a.PL = s->nx * s->ny;
    a.cstride = s->cstride;
    a.SI = s->cstride;  // SoA; the engine may switch to the row-blocked layout
    a.SZ = a.PL;
    a.SY = s->nx;
    a.nz_global = s->nzl;
    a.z0 = 0;
    if (p) {
        for (int i = 0; i < Q; ++i) {
            a.wv[i] = p->wv[i];
            a.lam[i] = p->lam[i];
        }
        a.cs2 = p->cs2;
        a.tau_f = p->tau_f;
        a.tau_g = p->tau_g;
        a.A = p->A;
        a.B = p->B;
        a.kappa = p->kappa;
        a.gamma = p->gamma;
        a.c1 = 2.0 * p->cs2;
        a.c2 = a.c1 * p->cs2;
        a.cs2sq = p->cs2 * p->cs2;
        a.srcpre = 1.0 - 0.5 / p->tau_f;
        for (int i = 0; i < Q; ++i) a.sw[i] = a.srcpre * a.wv[i];
        a.inv_tau_f = 1.0 / p->tau_f;
        a.inv_tau_g = 1.0 / p->tau_g;
        a.a1 = 1.0 / p->cs2;
        a.a2 = 1.0 / a.c2;
        a.a3 = 1.0 / a.c1;
        a.inv_cs2 = 1.0 / p->cs2;
        a.inv_cs2sq = 1.0 / a.cs2sq;
    }
}

static void set_planes(FluidArgs &a, int vvl, long long z_lo, long long z_hi) {
    a.z_lo = (int)z_lo;
    a.nplanes = (int)(z_hi - z_lo);
    a.nthreads = (long long)a.nplanes * a.ny * (a.nx / vvl);
}

static inline unsigned grid_for(long long n, int tpb) { return (unsigned)((n + tpb - 1) / tpb); }

constexpr int kTPB = 128;

static int launch_phi(const FluidArgs &a, int vvl, cudaStream_t st) {
    if (a.nthreads <= 0) return LTK_OK;
    const unsigned g = grid_for(a.nthreads, kTPB);
    switch (vvl) {
        case 1: k_phi<1><<<g, kTPB, 0, st>>>(a); break;
        case 2: k_phi<2><<<g, kTPB, 0, st>>>(a); break;
        default: k_phi<4><<<g, kTPB, 0, st>>>(a); break;
    }
    LTK_CHECK_LAUNCH("k_phi");
    return LTK_OK;
}

// mu stencil kernel (process-wide): LTK_MU_AUTO = k_mu_lds where it applies,
// else k_mu_tma, else k_mu; LTK_MU_COL / LTK_MU_BLK = k_mu_col / k_mu_blk in
// k_mu_lds's place; LTK_MU_TMA skips the 2.5-D kernels; LTK_MU_PLAIN = k_mu.
static int &mu_variant() {
    static int v = LTK_MU_AUTO;
    return v;
}

static int launch_mu(const FluidArgs &a, int vvl, cudaStream_t st) {
    if (a.nthreads <= 0) return LTK_OK;
    const int variant = mu_variant();
    if ((variant == LTK_MU_AUTO || variant == LTK_MU_COL || variant == LTK_MU_BLK) &&
        mu_col_ok(a)) {
        if (variant == LTK_MU_AUTO) {  // shared-memory tile filled by cp.async
            dim3 grid((unsigned)(a.nx / 32), (unsigned)(a.ny / 8),
                      (unsigned)((a.nplanes + kMuLdsZ - 1) / kMuLdsZ));
            k_mu_lds<kMuLdsZ><<<grid, dim3(32, 8), 0, st>>>(a);
            LTK_CHECK_LAUNCH("k_mu_lds");
            return LTK_OK;
        }
        if (variant == LTK_MU_BLK) {
            dim3 grid((unsigned)(a.nx / 32), (unsigned)(a.ny / 8),
                      (unsigned)((a.nplanes + kMuBlkZ - 1) / kMuBlkZ));
            k_mu_blk<kMuBlkZ><<<grid, dim3(32, 8), 0, st>>>(a);
            LTK_CHECK_LAUNCH("k_mu_blk");
            return LTK_OK;
        }
        dim3 grid((unsigned)(a.nx / 32), (unsigned)(a.ny / 8),
                  (unsigned)((a.nplanes + kMuColZ - 1) / kMuColZ));
        k_mu_col<><<<grid, dim3(32, 8), 0, st>>>(a);
        LTK_CHECK_LAUNCH("k_mu_col");
        return LTK_OK;
    }
    if (variant != LTK_MU_PLAIN && mu_tma_ok(a)) {
        // shared-memory staged stencil, rows loaded by TMA bulk copies
        static bool attr_set = false;
        if (!attr_set) {
            LTK_CUDA(cudaFuncSetAttribute(k_mu_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(200 * 1024)));
            LTK_CUDA(cudaFuncSetAttribute(k_mu_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(200 * 1024)));
            attr_set = true;
        }
        const int rows = mu_tma_rows(a.nx);
        dim3 grid((unsigned)(a.ny / rows), (unsigned)((a.nplanes + kMuZ - 1) / kMuZ));
        const int threads = std::min(256, (a.nx + 31) / 32 * 32);
        if (rows == 4)
            k_mu_tma<4><<<grid, threads, mu_tma_smem(a), st>>>(a);
        else
            k_mu_tma<2><<<grid, threads, mu_tma_smem(a), st>>>(a);
        LTK_CHECK_LAUNCH("k_mu_tma");
        return LTK_OK;
    }
    const unsigned g = grid_for(a.nthreads, kTPB);
    switch (vvl) {
        case 1: k_mu<1><<<g, kTPB, 0, st>>>(a); break;
        case 2: k_mu<2><<<g, kTPB, 0, st>>>(a); break;
        default: k_mu<4><<<g, kTPB, 0, st>>>(a); break;
    }
    LTK_CHECK_LAUNCH("k_mu");
    return LTK_OK;
}

// collide-stream kernel variant (process-wide): LTK_CS_REG register-resident
// k_collide_stream, LTK_CS_TMA TMA-staged k_cs_tma where it applies (nx a
// multiple of 128, VVL 1).  Default from env LTK_CS_VARIANT, else TMA.
static int &cs_variant() {
    static int v = getenv("LTK_CS_VARIANT") ? atoi(getenv("LTK_CS_VARIANT")) : LTK_CS_REG;
    return v;
}

static bool use_cs_tma(const FluidArgs &a, int vvl) {
    return cs_variant() == LTK_CS_TMA && cs_tma_ok(a, vvl);
}

template <int MODE, int PHYS, int T1>
static void launch_cs_t(const FluidArgs &a, int vvl, cudaStream_t st) {
    const unsigned g = grid_for(a.nthreads, kTPB);
    if (vvl == 2)
        k_collide_stream<2, MODE, PHYS, T1><<<g, kTPB, 0, st>>>(a);
    else
        k_collide_stream<1, MODE, PHYS, T1><<<g, kTPB, 0, st>>>(a);
}


template <int PHYS>
static void launch_cs_exact(const FluidArgs &a, int vvl, cudaStream_t st) {
    // x / 1.0 == x: skip the relaxation divisions when tau is exactly 1
    switch ((a.tau_f == 1.0 ? 1 : 0) | (a.tau_g == 1.0 ? 2 : 0)) {
        case 0: launch_cs_t<LTK_MODE_EXACT, PHYS, 0>(a, vvl, st); break;
        case 1: launch_cs_t<LTK_MODE_EXACT, PHYS, 1>(a, vvl, st); break;
        case 2: launch_cs_t<LTK_MODE_EXACT, PHYS, 2>(a, vvl, st); break;
        default: launch_cs_t<LTK_MODE_EXACT, PHYS, 3>(a, vvl, st); break;
    }
}

static int launch_cs(const FluidArgs &a, int vvl, int mode, int phys, cudaStream_t st) {
    if (a.nthreads <= 0) return LTK_OK;
    if (phys != 2 && use_cs_tma(a, vvl)) return launch_cs_tma(a, mode, phys, st);
    if (vvl > 2) return fail(LTK_ERR_PLAN, "collide-stream supports vvl 1, 2 (got %d)", vvl);
    if (phys == 2 && !a.aux) return fail(LTK_ERR_CONFIG, "stress form needs the engine's aux arrays");
    if (mode == LTK_MODE_EXACT && phys == 2) launch_cs_exact<2>(a, vvl, st);
    else if (mode == LTK_MODE_EXACT && phys == 1) launch_cs_exact<1>(a, vvl, st);
    else if (mode == LTK_MODE_EXACT) launch_cs_exact<0>(a, vvl, st);
    else if (phys == 2) launch_cs_t<LTK_MODE_FAST, 2, 0>(a, vvl, st);
    else if (phys == 1) launch_cs_t<LTK_MODE_FAST, 1, 0>(a, vvl, st);
    else launch_cs_t<LTK_MODE_FAST, 0, 0>(a, vvl, st);
    LTK_CHECK_LAUNCH("k_collide_stream");
    return LTK_OK;
}

// Fused collide-stream + next-state phi (k_cs_phi).  Collides planes
// [a.z_lo, a.z_lo + a.nplanes) and forms phi_next on [phi_lo, phi_hi), which
// must lie strictly inside the collided planes.  extra_lag: planes of slack
// between the collision front and the phi front beyond the 3 the
// no-deadlock argument needs (fluid_kernels.cuh).
static bool fuse_fields(FluidArgs &a, int vvl, int phi_lo, int phi_hi, int extra_lag,
                        unsigned long long *sync) {
    if (!sync || phi_hi <= phi_lo || phi_lo < a.z_lo + 1 || phi_hi > a.z_lo + a.nplanes - 1)
        return false;
    a.sync = sync;
    a.tpp = (long long)a.ny * (a.nx / vvl);
    a.phi_lo = phi_lo;
    a.phi_hi = phi_hi;
    // CTA b waits (before colliding) on planes up to phi plane + 1: they must
    // lie in tickets < b, i.e. lag_ctas*128 > (phi_lo - z_lo + 2) * tpp + 127
    const long long lag_threads = (long long)(phi_lo - a.z_lo + 2 + extra_lag) * a.tpp;
    a.lag_ctas = (unsigned)((lag_threads + kTPB - 1) / kTPB) + 1;
    a.ncta_cs = grid_for(a.nthreads, kTPB);
    const unsigned nphi = grid_for((long long)(phi_hi - phi_lo) * a.tpp, kTPB);
    a.ncta = std::max(a.ncta_cs, a.lag_ctas + nphi);
    return true;
}

// L2 policy of the fused kernel's state traffic (bit 0: evict-first input
// loads, bit 1: evict-first f' / evict-last g' stores); env LTK_FUSE_HINT.
static int fuse_hint() {
    static const int h = getenv("LTK_FUSE_HINT") ? atoi(getenv("LTK_FUSE_HINT")) & 3 : 2;
    return h;
}

template <int MODE, int PHYS, int T1, int H>
static void launch_csphi_h(const FluidArgs &a, int vvl, cudaStream_t st) {
    if (vvl == 2)
        k_cs_phi<2, MODE, PHYS, T1, H><<<a.ncta, kTPB, 0, st>>>(a);
    else
        k_cs_phi<1, MODE, PHYS, T1, H><<<a.ncta, kTPB, 0, st>>>(a);
}

template <int MODE, int PHYS, int T1>
static void launch_csphi_t(const FluidArgs &a, int vvl, cudaStream_t st) {
    switch (fuse_hint()) {
        case 0: launch_csphi_h<MODE, PHYS, T1, 0>(a, vvl, st); break;
        case 1: launch_csphi_h<MODE, PHYS, T1, 1>(a, vvl, st); break;
        case 2: launch_csphi_h<MODE, PHYS, T1, 2>(a, vvl, st); break;
        default: launch_csphi_h<MODE, PHYS, T1, 3>(a, vvl, st); break;
    }
}

template <int PHYS>
static void launch_csphi_exact(const FluidArgs &a, int vvl, cudaStream_t st) {
    switch ((a.tau_f == 1.0 ? 1 : 0) | (a.tau_g == 1.0 ? 2 : 0)) {
        case 0: launch_csphi_t<LTK_MODE_EXACT, PHYS, 0>(a, vvl, st); break;
        case 1: launch_csphi_t<LTK_MODE_EXACT, PHYS, 1>(a, vvl, st); break;
        case 2: launch_csphi_t<LTK_MODE_EXACT, PHYS, 2>(a, vvl, st); break;
        default: launch_csphi_t<LTK_MODE_EXACT, PHYS, 3>(a, vvl, st); break;
    }
}

static int launch_cs_phi(const FluidArgs &a, int vvl, int mode, int phys, cudaStream_t st) {
    if (a.nthreads <= 0) return LTK_OK;
    if (vvl > 2) return fail(LTK_ERR_PLAN, "collide-stream supports vvl 1, 2 (got %d)", vvl);
    if (mode == LTK_MODE_EXACT && phys == 1) launch_csphi_exact<1>(a, vvl, st);
    else if (mode == LTK_MODE_EXACT) launch_csphi_exact<0>(a, vvl, st);
    else if (phys == 1) launch_csphi_t<LTK_MODE_FAST, 1, 0>(a, vvl, st);
    else launch_csphi_t<LTK_MODE_FAST, 0, 0>(a, vvl, st);
    LTK_CHECK_LAUNCH("k_cs_phi");
    return LTK_OK;
}

// ------------------------------------------------------------------ plane copies
// Each copy moves `rows` rows of `row` doubles (row even), rows `stride`
// doubles apart on both sides; a contiguous plane is rows = 1, row = PL.
struct PlaneCopies {
    const double *src[24];
    double *dst[24];
    int n;
    long long PL;      // doubles per copy (rows * row)
    long long row = 0; // 0: contiguous (row = PL)
    long long stride = 0;
};

__global__ void __launch_bounds__(256) k_plane_copy(const PlaneCopies pc) {
    const int j = blockIdx.y;
    const double *s = pc.src[j];
    double *d = pc.dst[j];
    const long long n2 = pc.PL / 2;
    const long long r2 = pc.row / 2;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2;
         i += (long long)gridDim.x * blockDim.x) {
        long long o = 2 * i;
        if (r2) o = (i / r2) * pc.stride + 2 * (i % r2);
        *reinterpret_cast<double2 *>(d + o) = *reinterpret_cast<const double2 *>(s + o);
    }
}

static int run_plane_copies(const PlaneCopies &pc, cudaStream_t st) {
    if (pc.n == 0) return LTK_OK;
    dim3 grid((unsigned)std::min<long long>((pc.PL / 2 + 255) / 256, 148 * 4), pc.n);
    k_plane_copy<<<grid, 256, 0, st>>>(pc);
    LTK_CHECK_LAUNCH("k_plane_copy");
    return LTK_OK;
}

constexpr int kUp[5] = {5, 11, 13, 15, 17};    // cz = +1
constexpr int kDown[5] = {6, 12, 14, 16, 18};  // cz = -1

static inline double *plane(double *base, const ltk_slab *s, int comp, long long zs) {
    return base + comp * s->cstride + zs * s->nx * s->ny;
}

// f/g storage layout: element (comp i, storage plane zs, row y, x) at
// i*SI + zs*SZ + y*SY + x.  SoA (component-major planes) is the C-ABI slab
// layout; the engine may hold its state row-blocked instead (the 19
// components of one x-row adjacent), which keeps the pages a CTA touches at
// once few.
struct Lay {
    long long SI, SZ, SY;
};
static inline Lay soa_lay(const ltk_slab *s) { return {s->cstride, s->nx * s->ny, s->nx}; }
static inline Lay row_lay(const ltk_slab *s) { return {s->nx, s->ny * Q * s->nx, Q * s->nx}; }
static inline bool is_soa(const Lay &L, const ltk_slab *s) { return L.SY == s->nx && L.SI == s->cstride; }
static inline double *plane(double *base, const Lay &L, int comp, long long zs) {
    return base + comp * L.SI + zs * L.SZ;
}
// the copy geometry of one component plane in layout L
static inline void plane_geom(PlaneCopies &pc, const Lay &L, const ltk_slab *s) {
    pc.PL = s->nx * s->ny;
    if (L.SY == s->nx) {
        pc.row = pc.stride = 0;
    } else {
        pc.row = s->nx;
        pc.stride = L.SY;
    }
}

// ------------------------------------------------------------------ transposes
// host order site (x*ny + y)*nzg + z  <->  slab (z - z0 + 1)*PL + y*nx + x.
// 32x32 (x, z) tiles staged in shared memory, both sides coalesced.
template <bool TO_SLAB>
__global__ void __launch_bounds__(256) k_transpose(double *slab, double *host, long long nx,
                                                   long long ny, long long nzl, long long nzg,
                                                   long long z0, long long padded, long long SI,
                                                   long long SZ, long long SY, int ncomp) {
    __shared__ double tile[32][33];
    const int tx = threadIdx.x, ty = threadIdx.y;  // (32, 8)
    const long long xb = (long long)blockIdx.x * 32, zb = (long long)blockIdx.y * 32;
    const long long yc = blockIdx.z;
    const long long y = yc % ny;
    const int c = (int)(yc / ny);
    if (c >= ncomp) return;
    double *h = host + (long long)c * padded;
    double *sl = slab + (long long)c * SI + y * SY;
    if (TO_SLAB) {
        for (int k = ty; k < 32; k += 8) {  // read host: z fastest
            const long long x = xb + k, z = zb + tx;
            if (x < nx && z < nzl) tile[k][tx] = h[(x * ny + y) * nzg + z0 + z];
        }
        __syncthreads();
        for (int k = ty; k < 32; k += 8) {  // write slab: x fastest
            const long long x = xb + tx, z = zb + k;
            if (x < nx && z < nzl) sl[(z + 1) * SZ + x] = tile[tx][k];
        }
    } else {
        for (int k = ty; k < 32; k += 8) {
            const long long x = xb + tx, z = zb + k;
            if (x < nx && z < nzl) tile[tx][k] = sl[(z + 1) * SZ + x];
        }
        __syncthreads();
        for (int k = ty; k < 32; k += 8) {
            const long long x = xb + k, z = zb + tx;
            if (x < nx && z < nzl) h[(x * ny + y) * nzg + z0 + z] = tile[k][tx];
        }
    }
}

static int transpose(const ltk_slab *s, const Lay &L, double *slab, double *host,
                     long long padded, long long nzg, long long z0, int ncomp, bool to_slab,
                     cudaStream_t st) {
    if (z0 < 0 || z0 + s->nzl > nzg) return fail(LTK_ERR_SHAPE, "slab planes outside lattice");
    if (padded < s->nx * s->ny * nzg) return fail(LTK_ERR_SHAPE, "padded < nsites");
    if ((long long)s->ny * ncomp > 65535LL * 65535LL) return fail(LTK_ERR_SHAPE, "too many rows");
    dim3 block(32, 8);
    dim3 grid((unsigned)((s->nx + 31) / 32), (unsigned)((s->nzl + 31) / 32),
              (unsigned)(s->ny * ncomp));
    if (grid.z > 65535) return fail(LTK_ERR_SHAPE, "ny*ncomp exceeds 65535");
    if (to_slab)
        k_transpose<true><<<grid, block, 0, st>>>(slab, host, s->nx, s->ny, s->nzl, nzg, z0,
                                                  padded, L.SI, L.SZ, L.SY, ncomp);
    else
        k_transpose<false><<<grid, block, 0, st>>>(slab, host, s->nx, s->ny, s->nzl, nzg, z0,
                                                   padded, L.SI, L.SZ, L.SY, ncomp);
    LTK_CHECK_LAUNCH("k_transpose");
    return LTK_OK;
}

// ------------------------------------------------------------------ masked pack
__global__ void k_pack_sites(const double *src, double *packed, const long long *idx,
                             long long k, int ncomp, long long padded, int unpack) {
    const long long n = k * ncomp;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        const long long c = t / k, j = t - c * k;
        const long long e = c * padded + idx[j];
        if (unpack)
            const_cast<double *>(src)[e] = packed[t];
        else
            packed[t] = src[e];
    }
}

// ------------------------------------------------------------------ NCCL (dlopen)
struct Nccl {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
};

static Nccl &nccl() {
    static Nccl n;
    static bool tried = false;
    if (!tried) {
        tried = true;
        n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!n.h) n.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (n.h) {
            n.GetUniqueId = (decltype(n.GetUniqueId))dlsym(n.h, "ncclGetUniqueId");
            n.CommInitRank = (decltype(n.CommInitRank))dlsym(n.h, "ncclCommInitRank");
            n.CommDestroy = (decltype(n.CommDestroy))dlsym(n.h, "ncclCommDestroy");
            n.GroupStart = (decltype(n.GroupStart))dlsym(n.h, "ncclGroupStart");
            n.GroupEnd = (decltype(n.GroupEnd))dlsym(n.h, "ncclGroupEnd");
            n.Send = (decltype(n.Send))dlsym(n.h, "ncclSend");
            n.Recv = (decltype(n.Recv))dlsym(n.h, "ncclRecv");
            n.GetErrorString = (decltype(n.GetErrorString))dlsym(n.h, "ncclGetErrorString");
            n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.GroupStart &&
                   n.GroupEnd && n.Send && n.Recv && n.GetErrorString;
        }
    }
    return n;
}

#define LTK_NCCL(call)                                                                 \
    do {                                                                               \
        ncclResult_t r_ = (call);                                                      \
        if (r_ != ncclSuccess)                                                         \
            return fail(LTK_ERR_DEVICE, "%s: %s", #call, nccl().GetErrorString(r_));    \
    } while (0)

}  // namespace ltk

// ------------------------------------------------------------------ engine
struct ltk_fluid {
    int dev = 0;
    long long nx = 0, ny = 0, nzg = 0, nzl = 0, z0 = 0;
    int rank = 0, nranks = 1, vvl = 1;
    ltk_fluid_params prm{};
    ltk_slab slab{};
    ltk::Lay lay{};  // f/g layout (SoA unless ltk_fluid_set_layout / LTK_LAYOUT=1 chose row-blocked)
    double *fg[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [state][f/g]
    // phi per state in one allocation (phi of state s at phi + s*phi_stride):
    // the fused kernel forms the next state's phi while this step's stays
    double *phi = nullptr, *mu = nullptr;
    long long phi_stride = 0;
    int cur = 0;
    // fused collide-stream + phi (k_cs_phi): counters [nzl + 2]; phi planes of
    // the current state already formed by the previous step ([lo, hi))
    unsigned long long *fsync = nullptr;
    unsigned fuse_ncta = 0;  // grid of the fused launches counted in fsync
    bool fuse = false;  // measured slower than the three-kernel step
    bool peer_overlap = true;  // peer transport: boundary planes on comm_st (env LTK_PEER_OVERLAP)
    int fuse_lag = 1;
    int phi_lo = 0, phi_hi = 0;
    double *phi_of(int s) const { return phi + s * phi_stride; }
    cudaStream_t st = nullptr, comm_st = nullptr;
    cudaEvent_t ev_fork[3] = {}, ev_join[3] = {};
    ncclComm_t comm = nullptr;
    // transport between slabs: LOCAL (one slab, periodic images into itself),
    // NCCL (face exchanges on comm_st), PEER (CUDA IPC: halo images stored by
    // the kernels straight into the neighbours' buffers over NVLink)
    int transport = 0;
    struct Peer {
        double *fg[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
        double *phi[2] = {nullptr, nullptr}, *mu = nullptr;
        unsigned long long *inbox = nullptr;
    } up, dn;
    unsigned long long *inbox = nullptr;  // [2]: progress of the slab below / above
    int *peer_timeout = nullptr;
    std::vector<void *> ipc_opened;
    long long step = 0;   // timesteps taken (lockstep across slabs)
    bool primed = false;  // peer transport: halos re-primed by a load since the last step
    bool use_graph = false;
    cudaGraphExec_t gexec[4] = {nullptr, nullptr, nullptr, nullptr};  // [state + 2*(phi formed)]
    int gnxt[4][2] = {};  // phi planes each graph's step forms
    bool prof = false;
    cudaEvent_t pev[5] = {};          // events of the step being enqueued
    std::vector<cudaEvent_t> ppool;   // 4 per profiled step, read at the end
    long long prof_steps = 0;
};

namespace ltk {

static void drop_graphs(ltk_fluid *e) {
    for (auto &g : e->gexec)
        if (g) {
            cudaGraphExecDestroy(g);
            g = nullptr;
        }
}

enum { kLocal = 0, kNccl = 1, kPeer = 2 };

static FluidArgs engine_args(const ltk_fluid *e, int in_state) {
    FluidArgs a;
    fill_args(a, &e->slab, &e->prm);
    a.nz_global = e->nzg;
    a.z0 = e->z0;
    a.SI = e->lay.SI;
    a.SZ = e->lay.SZ;
    a.SY = e->lay.SY;
    a.f_in = e->fg[in_state][0];
    a.g_in = e->fg[in_state][1];
    a.f_out = e->fg[1 - in_state][0];
    a.g_out = e->fg[1 - in_state][1];
    a.phi_in = e->phi_of(in_state);
    a.phi_out = e->phi_of(in_state);
    a.phi_next = e->phi_of(1 - in_state);
    a.mu = e->mu;
    a.mu_out = e->mu;
    a.astride = e->phi_stride;
    a.aux = e->prm.physics == 2 ? e->mu + e->phi_stride : nullptr;  // after mu, same allocation
    a.err = singular_word();
    if (e->transport == kLocal) {  // periodic images into this slab
        a.img_f_up = a.img_f_dn = a.f_out;
        a.img_g_up = a.img_g_dn = a.g_out;
        a.img_phi_up = a.img_phi_dn = e->phi_of(in_state);
        a.img_mu_up = a.img_mu_dn = e->mu;
        a.img_aux_up = a.img_aux_dn = a.aux;
    } else if (e->transport == kPeer) {  // images into the neighbours over NVLink
        a.img_f_up = e->up.fg[1 - in_state][0];
        a.img_g_up = e->up.fg[1 - in_state][1];
        a.img_f_dn = e->dn.fg[1 - in_state][0];
        a.img_g_dn = e->dn.fg[1 - in_state][1];
        a.img_phi_up = e->up.phi[in_state];
        a.img_phi_dn = e->dn.phi[in_state];
        a.img_mu_up = e->up.mu;
        a.img_mu_dn = e->dn.mu;
        if (a.aux) {  // peers share the layout: their aux follows their mu
            a.img_aux_up = e->up.mu + e->phi_stride;
            a.img_aux_dn = e->dn.mu + e->phi_stride;
        }
    }
    return a;
}

// One NCCL halo exchange group on comm_st.  kind 0: f/g crossing components
// of state `s`; kind 1: phi; kind 2: mu.  Send order per peer is fixed
// (faces up, then faces down) and receive order mirrors it, which keeps the
// matching right even when both neighbours are the same rank (P = 2) or
// this rank itself (P = 1).
static int exchange(ltk_fluid *e, int kind, int s) {
    Nccl &n = nccl();
    const int up = (e->rank + 1) % e->nranks, down = (e->rank + e->nranks - 1) % e->nranks;
    const size_t PL = (size_t)(e->nx * e->ny);
    const long long top = e->nzl, bot = 1, halo_lo = 0, halo_hi = e->nzl + 1;
    const ltk_slab *sl = &e->slab;
    LTK_NCCL(n.GroupStart());
    if (kind == 0) {
        for (int d = 0; d < 2; ++d)
            for (int j = 0; j < 5; ++j)
                LTK_NCCL(n.Send(plane(e->fg[s][d], sl, kUp[j], top), PL, ncclFloat64, up, e->comm,
                                e->comm_st));
        for (int d = 0; d < 2; ++d)
            for (int j = 0; j < 5; ++j)
                LTK_NCCL(n.Send(plane(e->fg[s][d], sl, kDown[j], bot), PL, ncclFloat64, down,
                                e->comm, e->comm_st));
        for (int d = 0; d < 2; ++d)
            for (int j = 0; j < 5; ++j)
                LTK_NCCL(n.Recv(plane(e->fg[s][d], sl, kUp[j], halo_lo), PL, ncclFloat64, down,
                                e->comm, e->comm_st));
        for (int d = 0; d < 2; ++d)
            for (int j = 0; j < 5; ++j)
                LTK_NCCL(n.Recv(plane(e->fg[s][d], sl, kDown[j], halo_hi), PL, ncclFloat64, up,
                                e->comm, e->comm_st));
    } else {
        // kind 1: phi; kind 2: mu, and for the stress form the 4 aux arrays after it
        const int nb = (kind == 2 && e->prm.physics == 2) ? 5 : 1;
        for (int k = 0; k < nb; ++k) {
            double *b = (kind == 1 ? e->phi_of(s) : e->mu) + (long long)k * e->phi_stride;
            LTK_NCCL(n.Send(b + top * PL, PL, ncclFloat64, up, e->comm, e->comm_st));
            LTK_NCCL(n.Send(b + bot * PL, PL, ncclFloat64, down, e->comm, e->comm_st));
        }
        for (int k = 0; k < nb; ++k) {
            double *b = (kind == 1 ? e->phi_of(s) : e->mu) + (long long)k * e->phi_stride;
            LTK_NCCL(n.Recv(b + halo_lo * PL, PL, ncclFloat64, down, e->comm, e->comm_st));
            LTK_NCCL(n.Recv(b + halo_hi * PL, PL, ncclFloat64, up, e->comm, e->comm_st));
        }
    }
    LTK_NCCL(n.GroupEnd());
    return LTK_OK;
}

#define LTK_RC(x)              \
    do {                       \
        int rc_ = (x);         \
        if (rc_) return rc_;   \
    } while (0)

static int enqueue_step_peer(ltk_fluid *e, int s, cudaStream_t st, bool prof, int nxt[2]);

// phi of state s on planes [lo, hi) minus those the previous step's fused
// kernel already formed ([e->phi_lo, e->phi_hi)).
template <class L>
static int phi_rest(ltk_fluid *e, FluidArgs &a, long long lo, long long hi, L launch_one) {
    const int vvl = e->vvl;
    const long long dlo = std::max(lo, std::min(hi, (long long)e->phi_lo));
    const long long dhi = std::max(dlo, std::min(hi, (long long)e->phi_hi));
    if (dlo > lo) {
        set_planes(a, vvl, lo, dlo);
        LTK_RC(launch_one());
    }
    if (hi > dhi) {
        set_planes(a, vvl, dhi, hi);
        LTK_RC(launch_one());
    }
    return LTK_OK;
}

// Collide-stream of planes [lo, hi): fused with the next state's phi on
// [lo + 1, hi - 1) when enabled and long enough, else the plain kernel.
// nxt receives the phi planes formed.
static int cs_planes(ltk_fluid *e, FluidArgs &a, long long lo, long long hi, cudaStream_t st,
                     int nxt[2]) {
    const int vvl = e->vvl, mode = e->prm.mode, phys = e->prm.physics;
    if (hi <= lo) return LTK_OK;
    set_planes(a, vvl, lo, hi);
    if (e->fuse && e->prm.physics != 2 && a.ny * (a.nx / vvl) >= kTPB &&
        fuse_fields(a, vvl, (int)lo + 1, (int)hi - 1, e->fuse_lag, e->fsync)) {
        if (a.ncta != e->fuse_ncta) {  // launch epochs are ticket / ncta: restart the count
            LTK_CUDA(cudaMemsetAsync(e->fsync, 0, (size_t)(e->nzl + 1) * 8, st));
            e->fuse_ncta = a.ncta;
        }
        LTK_RC(launch_cs_phi(a, vvl, mode, phys, st));
        nxt[0] = (int)lo + 1;
        nxt[1] = (int)hi - 1;
        return LTK_OK;
    }
    return launch_cs(a, vvl, mode, phys, st);
}

// Enqueue one timestep reading state `s` and writing state 1 - s.  nxt: the
// phi planes of state 1 - s formed on the way (by the fused kernel).
static int enqueue_step(ltk_fluid *e, int s, cudaStream_t st, bool prof, int nxt[2]) {
    FluidArgs a = engine_args(e, s);
    const int vvl = e->vvl, mode = e->prm.mode, phys = e->prm.physics;
    const long long nzl = e->nzl;
    nxt[0] = nxt[1] = 0;
    if (e->transport == kPeer) return enqueue_step_peer(e, s, st, prof, nxt);
    auto phi = [&] { return launch_phi(a, vvl, st); };
    if (prof) cudaEventRecord(e->pev[0], st);
    if (e->transport == kLocal) {
        // single slab, periodic z: halos written by the kernels; phi of the
        // interior planes came with the previous step's collide-stream
        LTK_RC(phi_rest(e, a, 0, nzl, phi));
        if (prof) cudaEventRecord(e->pev[1], st);
        if (phys >= 1) {
            set_planes(a, vvl, 0, nzl);
            LTK_RC(launch_mu(a, vvl, st));
        }
        if (prof) cudaEventRecord(e->pev[2], st);
        LTK_RC(cs_planes(e, a, 0, nzl, st, nxt));
        if (prof) cudaEventRecord(e->pev[3], st);
        return LTK_OK;
    }
    // z-slabs: each exchange overlaps the interior planes of the next kernel
    const long long in_lo = 1, in_hi = nzl - 1;  // interior (may be empty)
    auto boundary = [&](auto launch_one) -> int {
        set_planes(a, vvl, 0, 1);
        LTK_RC(launch_one());
        if (nzl > 1) {
            set_planes(a, vvl, nzl - 1, nzl);
            LTK_RC(launch_one());
        }
        return LTK_OK;
    };
    // (1) f/g faces || phi interior
    LTK_CUDA(cudaEventRecord(e->ev_fork[0], st));
    LTK_CUDA(cudaStreamWaitEvent(e->comm_st, e->ev_fork[0], 0));
    LTK_RC(exchange(e, 0, s));
    LTK_CUDA(cudaEventRecord(e->ev_join[0], e->comm_st));
    if (in_hi > in_lo) LTK_RC(phi_rest(e, a, in_lo, in_hi, phi));
    LTK_CUDA(cudaStreamWaitEvent(st, e->ev_join[0], 0));
    LTK_RC(boundary(phi));
    if (prof) cudaEventRecord(e->pev[1], st);
    if (phys >= 1) {
        // (2) phi faces || mu interior
        LTK_CUDA(cudaEventRecord(e->ev_fork[1], st));
        LTK_CUDA(cudaStreamWaitEvent(e->comm_st, e->ev_fork[1], 0));
        LTK_RC(exchange(e, 1, s));
        LTK_CUDA(cudaEventRecord(e->ev_join[1], e->comm_st));
        if (in_hi > in_lo) {
            set_planes(a, vvl, in_lo, in_hi);
            LTK_RC(launch_mu(a, vvl, st));
        }
        LTK_CUDA(cudaStreamWaitEvent(st, e->ev_join[1], 0));
        LTK_RC(boundary([&] { return launch_mu(a, vvl, st); }));
        // (3) mu faces || collide-stream interior
        LTK_CUDA(cudaEventRecord(e->ev_fork[2], st));
        LTK_CUDA(cudaStreamWaitEvent(e->comm_st, e->ev_fork[2], 0));
        LTK_RC(exchange(e, 2, s));
        LTK_CUDA(cudaEventRecord(e->ev_join[2], e->comm_st));
    }
    if (prof) cudaEventRecord(e->pev[2], st);
    LTK_RC(cs_planes(e, a, in_lo, in_hi, st, nxt));
    if (phys >= 1) LTK_CUDA(cudaStreamWaitEvent(st, e->ev_join[2], 0));
    LTK_RC(boundary([&] { return launch_cs(a, vvl, mode, phys, st); }));
    if (prof) cudaEventRecord(e->pev[3], st);
    return LTK_OK;
}

// ---- diagnostics: totals of rho, momentum, phi over the owned sites
// Block partial sums in a fixed tree, summed on the host in block order:
// deterministic for a given lattice (not the numpy summation order).
constexpr int kTotBlocks = 592, kTotThreads = 256;

__global__ void __launch_bounds__(kTotThreads) k_totals(const double *f, const double *g,
                                                        long long nx, long long ny, long long nzl,
                                                        long long SI, long long SZ, long long SY,
                                                        double *partial) {
    const long long PL = nx * ny, n = PL * nzl;
    double acc[5] = {0, 0, 0, 0, 0};
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        const long long z = t / PL, r = t - z * PL, y = r / nx;
        const long long o = (z + 1) * SZ + y * SY + (r - y * nx);  // storage plane 1 onwards
        static_for<0, Q>([&](auto I) {
            const double fi = f[I.value * SI + o];
            acc[0] += fi;
            if constexpr (cx(I.value) != 0) acc[1] += cx(I.value) * fi;
            if constexpr (cy(I.value) != 0) acc[2] += cy(I.value) * fi;
            if constexpr (cz(I.value) != 0) acc[3] += cz(I.value) * fi;
            acc[4] += g[I.value * SI + o];
        });
    }
    __shared__ double red[5][kTotThreads];
    for (int k = 0; k < 5; ++k) red[k][threadIdx.x] = acc[k];
    __syncthreads();
    for (int w = kTotThreads / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w)
            for (int k = 0; k < 5; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x < 5) partial[blockIdx.x * 5 + threadIdx.x] = red[threadIdx.x][0];
}

// ---- peer transport: progress counters pushed into the neighbours' inboxes
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__global__ void k_peer_signal(unsigned long long *up_slot, unsigned long long *dn_slot,
                              unsigned long long v) {
    __threadfence_system();  // this slab's earlier peer stores before the counter
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(up_slot), "l"(v) : "memory");
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dn_slot), "l"(v) : "memory");
}

__global__ void k_peer_wait(const unsigned long long *inbox, unsigned long long target,
                            int *timeout) {
    long long spins = 0;
    while (ld_acquire_sys(inbox) < target || ld_acquire_sys(inbox + 1) < target) {
        if (++spins > (1LL << 25)) {  // never hang the GPU (~10 s): record and go on
            atomicExch(timeout, 1);
            break;
        }
        __nanosleep(256);
    }
}

static int peer_signal(ltk_fluid *e, unsigned long long v, cudaStream_t st) {
    // I am the lower neighbour of `up` (its inbox[0]) and the upper one of `dn` (inbox[1])
    k_peer_signal<<<1, 1, 0, st>>>(e->up.inbox, e->dn.inbox + 1, v);
    LTK_CHECK_LAUNCH("k_peer_signal");
    return LTK_OK;
}

static int peer_wait(ltk_fluid *e, unsigned long long target, cudaStream_t st) {
    k_peer_wait<<<1, 1, 0, st>>>(e->inbox, target, e->peer_timeout);
    LTK_CHECK_LAUNCH("k_peer_wait");
    return LTK_OK;
}

// One timestep with the peer transport.  Counter protocol per step t (each
// slab pushes its counter into the neighbours' inboxes; waits are ">="):
//   4t+1  f/g halo images of state t re-primed after a load (peer_prime)
//   4t+2  phi images sent      4t+3  mu images sent
//   4t+4  f/g images of state t+1 sent (= "state t+1 ready", 4(t+1))
// Every wait sits behind the interior planes of a kernel, so the neighbours'
// progress overlaps local work; the boundary planes then store their halo
// images straight into the neighbours over NVLink.
static int enqueue_step_peer(ltk_fluid *e, int s, cudaStream_t st, bool prof, int nxt[2]) {
    FluidArgs a = engine_args(e, s);
    const int vvl = e->vvl, mode = e->prm.mode, phys = e->prm.physics;
    const long long nzl = e->nzl;
    const unsigned long long t4 = 4ULL * (unsigned long long)e->step;
    // Boundary planes on a second stream (bs): a phase's boundary planes need the
    // neighbours' halos and the previous phase, never this phase's interior, so
    // progress wait + boundary kernels (with their peer stores) + signal run
    // concurrently with the interior kernel; the streams join before the next
    // phase.  overlap off: everything in order on st.
    cudaStream_t bs = e->peer_overlap ? e->comm_st : st;
    auto ranges = [&](long long lo, long long hi, auto launch_one) -> int {
        if (hi > lo) {
            set_planes(a, vvl, lo, hi);
            return launch_one();
        }
        return LTK_OK;
    };
    auto boundary = [&](auto launch_one) -> int {
        LTK_RC(ranges(0, 1, launch_one));
        if (nzl > 1) LTK_RC(ranges(nzl - 1, nzl, launch_one));
        return LTK_OK;
    };
    auto fork = [&](int k) -> int {
        if (bs == st) return LTK_OK;
        LTK_CUDA(cudaEventRecord(e->ev_fork[k], st));
        LTK_CUDA(cudaStreamWaitEvent(bs, e->ev_fork[k], 0));
        return LTK_OK;
    };
    auto join = [&](int k) -> int {
        if (bs == st) return LTK_OK;
        LTK_CUDA(cudaEventRecord(e->ev_join[k], bs));
        LTK_CUDA(cudaStreamWaitEvent(st, e->ev_join[k], 0));
        return LTK_OK;
    };
    auto phi_a = [&] { return launch_phi(a, vvl, st); };
    auto phi_b = [&] { return launch_phi(a, vvl, bs); };
    auto mu_a = [&] { return launch_mu(a, vvl, st); };
    auto mu_b = [&] { return launch_mu(a, vvl, bs); };
    auto cs_b = [&] { return launch_cs(a, vvl, mode, phys, bs); };
    if (prof) cudaEventRecord(e->pev[0], st);
    // phi: interior || (f/g halos of state s -> boundary planes -> signal 4t+2)
    LTK_RC(fork(0));
    LTK_RC(peer_wait(e, t4 + (e->primed ? 1 : 0), bs));
    e->primed = false;
    LTK_RC(boundary(phi_b));
    LTK_RC(peer_signal(e, t4 + 2, bs));
    if (nzl > 2) LTK_RC(phi_rest(e, a, 1, nzl - 1, phi_a));
    LTK_RC(join(0));
    if (prof) cudaEventRecord(e->pev[1], st);
    // mu: interior || (phi halos -> boundary planes) ; signal 4t+3
    LTK_RC(fork(1));
    if (phys >= 1) {
        LTK_RC(peer_wait(e, t4 + 2, bs));
        LTK_RC(boundary(mu_b));
    }
    LTK_RC(peer_signal(e, t4 + 3, bs));
    if (phys >= 1) LTK_RC(ranges(1, nzl - 1, mu_a));
    LTK_RC(join(1));
    if (prof) cudaEventRecord(e->pev[2], st);
    // collide-stream: interior || (mu halos -> boundary planes -> signal 4t+4)
    LTK_RC(fork(2));
    LTK_RC(peer_wait(e, t4 + 3, bs));
    LTK_RC(boundary(cs_b));
    LTK_RC(peer_signal(e, t4 + 4, bs));
    LTK_RC(cs_planes(e, a, 1, nzl - 1, st, nxt));
    LTK_RC(join(2));
    if (prof) cudaEventRecord(e->pev[3], st);
    return LTK_OK;
}

// Before a load with the peer transport: the neighbours must have finished
// the previous step (their reads of the halos we are about to re-prime).
static int peer_before_load(ltk_fluid *e, cudaStream_t st) {
    return peer_wait(e, 4ULL * (unsigned long long)e->step, st);
}

// After the load: push the crossing components of the owned boundary planes
// of state `s` into the neighbours' halos, then signal 4t+1.
static int peer_prime(ltk_fluid *e, int s, cudaStream_t st) {
    PlaneCopies pc;
    memset(&pc, 0, sizeof pc);
    plane_geom(pc, e->lay, &e->slab);
    const Lay &L = e->lay;
    for (int j = 0; j < 5; ++j)
        for (int d = 0; d < 2; ++d) {
            pc.src[pc.n] = plane(e->fg[s][d], L, kUp[j], e->nzl);
            pc.dst[pc.n++] = plane(e->up.fg[s][d], L, kUp[j], 0);
            pc.src[pc.n] = plane(e->fg[s][d], L, kDown[j], 1);
            pc.dst[pc.n++] = plane(e->dn.fg[s][d], L, kDown[j], e->nzl + 1);
        }
    LTK_RC(run_plane_copies(pc, st));
    e->primed = true;
    return peer_signal(e, 4ULL * (unsigned long long)e->step + 1, st);
}

// Load every kernel a step can launch.  With lazy module loading (the CUDA 12
// default) the first launch of a kernel loads its module, which waits for the
// device to go idle; with the peer transport a progress-wait kernel may be
// spinning on a neighbour whose work is not enqueued yet, so a lazy load in
// the middle of an enqueue would stall until the spin budget runs out.
template <int MODE, int PHYS, int T1>
static void preload_cs_t(cudaFuncAttributes &fa) {
    cudaFuncGetAttributes(&fa, k_collide_stream<1, MODE, PHYS, T1>);
    cudaFuncGetAttributes(&fa, k_collide_stream<2, MODE, PHYS, T1>);
    cudaFuncGetAttributes(&fa, k_cs_phi<1, MODE, PHYS, T1, 0>);
    cudaFuncGetAttributes(&fa, k_cs_phi<1, MODE, PHYS, T1, 1>);
    cudaFuncGetAttributes(&fa, k_cs_phi<1, MODE, PHYS, T1, 2>);
    cudaFuncGetAttributes(&fa, k_cs_phi<1, MODE, PHYS, T1, 3>);
    cudaFuncGetAttributes(&fa, k_cs_phi<2, MODE, PHYS, T1, 0>);
    cudaFuncGetAttributes(&fa, k_cs_phi<2, MODE, PHYS, T1, 1>);
    cudaFuncGetAttributes(&fa, k_cs_phi<2, MODE, PHYS, T1, 2>);
    cudaFuncGetAttributes(&fa, k_cs_phi<2, MODE, PHYS, T1, 3>);
}

template <int MODE, int PHYS>
static void preload_cs(cudaFuncAttributes &fa) {
    preload_cs_t<MODE, PHYS, 0>(fa);
    if constexpr (MODE == LTK_MODE_EXACT) {
        preload_cs_t<MODE, PHYS, 1>(fa);
        preload_cs_t<MODE, PHYS, 2>(fa);
        preload_cs_t<MODE, PHYS, 3>(fa);
    }
}

static int preload_step_kernels() {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_phi<1>);
    cudaFuncGetAttributes(&fa, k_phi<2>);
    cudaFuncGetAttributes(&fa, k_phi<4>);
    cudaFuncGetAttributes(&fa, k_mu<1>);
    cudaFuncGetAttributes(&fa, k_mu<2>);
    cudaFuncGetAttributes(&fa, k_mu<4>);
    cudaFuncGetAttributes(&fa, k_mu_col<>);
    cudaFuncGetAttributes(&fa, k_mu_blk<kMuBlkZ>);
    cudaFuncGetAttributes(&fa, k_mu_lds<kMuLdsZ>);
    cudaFuncGetAttributes(&fa, k_mu_tma<4>);
    cudaFuncGetAttributes(&fa, k_mu_tma<2>);
    cudaFuncGetAttributes(&fa, k_plane_copy);
    cudaFuncGetAttributes(&fa, k_peer_wait);
    cudaFuncGetAttributes(&fa, k_peer_signal);
    cudaFuncGetAttributes(&fa, k_transpose<true>);
    cudaFuncGetAttributes(&fa, k_transpose<false>);
    preload_cs<LTK_MODE_EXACT, 0>(fa);
    preload_cs<LTK_MODE_EXACT, 1>(fa);
    preload_cs<LTK_MODE_FAST, 0>(fa);
    preload_cs<LTK_MODE_FAST, 1>(fa);
    // stress form: register collide-stream only (no fused / TMA variants)
    cudaFuncGetAttributes(&fa, k_collide_stream<1, LTK_MODE_FAST, 2, 0>);
    cudaFuncGetAttributes(&fa, k_collide_stream<2, LTK_MODE_FAST, 2, 0>);
    for (auto k : {k_collide_stream<1, LTK_MODE_EXACT, 2, 0>, k_collide_stream<1, LTK_MODE_EXACT, 2, 1>,
                   k_collide_stream<1, LTK_MODE_EXACT, 2, 2>, k_collide_stream<1, LTK_MODE_EXACT, 2, 3>,
                   k_collide_stream<2, LTK_MODE_EXACT, 2, 0>, k_collide_stream<2, LTK_MODE_EXACT, 2, 1>,
                   k_collide_stream<2, LTK_MODE_EXACT, 2, 2>, k_collide_stream<2, LTK_MODE_EXACT, 2, 3>})
        cudaFuncGetAttributes(&fa, k);
    LTK_CUDA(cudaFuncSetAttribute(k_mu_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(200 * 1024)));
    LTK_CUDA(cudaFuncSetAttribute(k_mu_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(200 * 1024)));
    LTK_CUDA(cudaGetLastError());
    return LTK_OK;
}

static int wrap_state_halos(ltk_fluid *e, int s, int which, cudaStream_t st) {
    if (is_soa(e->lay, &e->slab))
        return ltk_fluid_wrap_halos(&e->slab, e->fg[s][0], e->fg[s][1], e->phi_of(s), e->mu,
                                    which, st);
    if (which & 1) {  // row-blocked f/g: the crossing components' periodic images
        PlaneCopies pc;
        memset(&pc, 0, sizeof pc);
        plane_geom(pc, e->lay, &e->slab);
        for (int j = 0; j < 5; ++j)
            for (int d = 0; d < 2; ++d) {
                double *b = e->fg[s][d];
                pc.src[pc.n] = plane(b, e->lay, kUp[j], e->nzl);
                pc.dst[pc.n++] = plane(b, e->lay, kUp[j], 0);
                pc.src[pc.n] = plane(b, e->lay, kDown[j], 1);
                pc.dst[pc.n++] = plane(b, e->lay, kDown[j], e->nzl + 1);
            }
        LTK_RC(run_plane_copies(pc, st));
    }
    if (which & 6)
        return ltk_fluid_wrap_halos(&e->slab, e->fg[s][0], e->fg[s][1], e->phi_of(s), e->mu,
                                    which & 6, st);
    return LTK_OK;
}

}  // namespace ltk

using namespace ltk;

extern "C" {

int ltk_fluid_phi(const ltk_slab *s, const double *g, double *phi, int64_t z_lo, int64_t z_hi,
                  void *stream) {
    LTK_RC(check_slab(s, 1));
    if (z_lo < 0 || z_hi > s->nzl || z_hi < z_lo) return fail(LTK_ERR_BOUNDS, "plane range");
    FluidArgs a;
    fill_args(a, s, nullptr);
    a.g_in = g;
    a.phi_out = phi;
    set_planes(a, 1, z_lo, z_hi);
    return launch_phi(a, 1, as_stream(stream));
}

int ltk_fluid_mu(const ltk_slab *s, const double *phi, double *mu, const ltk_fluid_params *p,
                 int64_t z_lo, int64_t z_hi, void *stream) {
    LTK_RC(check_slab(s, 1));
    if (z_lo < 0 || z_hi > s->nzl || z_hi < z_lo) return fail(LTK_ERR_BOUNDS, "plane range");
    FluidArgs a;
    fill_args(a, s, p);
    a.phi_in = phi;
    a.mu_out = mu;
    set_planes(a, 1, z_lo, z_hi);
    return launch_mu(a, 1, as_stream(stream));
}

int ltk_fluid_collide_stream(const ltk_slab *s, const double *f_in, const double *g_in,
                             const double *mu, double *f_out, double *g_out,
                             const ltk_fluid_params *p, int64_t z_lo, int64_t z_hi, int32_t vvl,
                             void *stream) {
    LTK_RC(check_slab(s, vvl));
    if (!p) return fail(LTK_ERR_CONFIG, "null params");
    if (z_lo < 0 || z_hi > s->nzl || z_hi < z_lo) return fail(LTK_ERR_BOUNDS, "plane range");
    FluidArgs a;
    fill_args(a, s, p);
    a.f_in = f_in;
    a.g_in = g_in;
    a.mu = mu;
    a.f_out = f_out;
    a.g_out = g_out;
    a.err = singular_word();
    set_planes(a, vvl, z_lo, z_hi);
    return launch_cs(a, vvl, p->mode, p->physics, as_stream(stream));
}

int ltk_fluid_wrap_halos(const ltk_slab *s, double *f, double *g, double *phi, double *mu,
                         int32_t which, void *stream) {
    LTK_RC(check_slab(s, 1));
    PlaneCopies pc;
    memset(&pc, 0, sizeof pc);
    pc.PL = s->nx * s->ny;
    const long long nzl = s->nzl;
    if (which & 1) {
        for (int j = 0; j < 5; ++j) {
            for (double *b : {f, g}) {
                pc.src[pc.n] = plane(b, s, kUp[j], nzl);
                pc.dst[pc.n++] = plane(b, s, kUp[j], 0);
                pc.src[pc.n] = plane(b, s, kDown[j], 1);
                pc.dst[pc.n++] = plane(b, s, kDown[j], nzl + 1);
            }
        }
    }
    for (int k = 0; k < 2; ++k) {
        double *b = k == 0 ? phi : mu;
        if (!(which & (2 << k)) || !b) continue;
        pc.src[pc.n] = b + nzl * pc.PL;
        pc.dst[pc.n++] = b;
        pc.src[pc.n] = b + pc.PL;
        pc.dst[pc.n++] = b + (nzl + 1) * pc.PL;
    }
    return run_plane_copies(pc, as_stream(stream));
}

int ltk_fluid_pack_face(const ltk_slab *s, const double *f, const double *g, double *buf,
                        int32_t dir, void *stream) {
    LTK_RC(check_slab(s, 1));
    if (dir != 1 && dir != -1) return fail(LTK_ERR_CONFIG, "dir must be +1 or -1");
    PlaneCopies pc;
    memset(&pc, 0, sizeof pc);
    pc.PL = s->nx * s->ny;
    const int *comps = dir > 0 ? kUp : kDown;
    const long long zs = dir > 0 ? s->nzl : 1;
    for (int d = 0; d < 2; ++d)
        for (int j = 0; j < 5; ++j) {
            pc.src[pc.n] = plane(const_cast<double *>(d ? g : f), s, comps[j], zs);
            pc.dst[pc.n] = buf + (long long)pc.n * pc.PL;
            ++pc.n;
        }
    return run_plane_copies(pc, as_stream(stream));
}

int ltk_fluid_unpack_face(const ltk_slab *s, double *f, double *g, const double *buf,
                          int32_t dir, void *stream) {
    LTK_RC(check_slab(s, 1));
    if (dir != 1 && dir != -1) return fail(LTK_ERR_CONFIG, "dir must be +1 or -1");
    PlaneCopies pc;
    memset(&pc, 0, sizeof pc);
    pc.PL = s->nx * s->ny;
    const int *comps = dir > 0 ? kUp : kDown;
    const long long zs = dir > 0 ? 0 : s->nzl + 1;
    for (int d = 0; d < 2; ++d)
        for (int j = 0; j < 5; ++j) {
            pc.src[pc.n] = buf + (long long)pc.n * pc.PL;
            pc.dst[pc.n] = plane(d ? g : f, s, comps[j], zs);
            ++pc.n;
        }
    return run_plane_copies(pc, as_stream(stream));
}

int ltk_fluid_scatter(const ltk_slab *s, const double *host, int64_t padded, int64_t nz_global,
                      int64_t z0, int32_t ncomp, double *slab, void *stream) {
    LTK_RC(check_slab(s, 1));
    return transpose(s, soa_lay(s), slab, const_cast<double *>(host), padded, nz_global, z0, ncomp, true,
                     as_stream(stream));
}

int ltk_fluid_gather(const ltk_slab *s, const double *slab, int64_t padded, int64_t nz_global,
                     int64_t z0, int32_t ncomp, double *host, void *stream) {
    LTK_RC(check_slab(s, 1));
    return transpose(s, soa_lay(s), const_cast<double *>(slab), host, padded, nz_global, z0, ncomp, false,
                     as_stream(stream));
}

int ltk_pack_sites(const double *src, double *packed, const int64_t *idx, int64_t k,
                   int32_t ncomp, int64_t padded, void *stream) {
    if (k <= 0) return LTK_OK;
    const long long n = k * ncomp;
    const unsigned g = (unsigned)std::min<long long>((n + 255) / 256, 148LL * 16);
    k_pack_sites<<<g, 256, 0, as_stream(stream)>>>(src, packed, (const long long *)idx, k, ncomp,
                                                   padded, 0);
    LTK_CHECK_LAUNCH("k_pack_sites");
    return LTK_OK;
}

int ltk_unpack_sites(double *dst, const double *packed, const int64_t *idx, int64_t k,
                     int32_t ncomp, int64_t padded, void *stream) {
    if (k <= 0) return LTK_OK;
    const long long n = k * ncomp;
    const unsigned g = (unsigned)std::min<long long>((n + 255) / 256, 148LL * 16);
    k_pack_sites<<<g, 256, 0, as_stream(stream)>>>(dst, const_cast<double *>(packed),
                                                   (const long long *)idx, k, ncomp, padded, 1);
    LTK_CHECK_LAUNCH("k_unpack_sites");
    return LTK_OK;
}

// ---------------------------------------------------------------- engine API

int ltk_fluid_create(int64_t nx, int64_t ny, int64_t nz_global, int32_t rank, int32_t nranks,
                     const ltk_fluid_params *p, int32_t vvl, ltk_fluid **out) {
    *out = nullptr;
    if (!p) return fail(LTK_ERR_CONFIG, "null params");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(LTK_ERR_CONFIG, "bad rank/nranks");
    if (nz_global % nranks)
        return fail(LTK_ERR_SHAPE, "nz %lld not divisible by %d ranks", (long long)nz_global,
                    nranks);
    if (p->tau_f <= 0.5 || p->tau_g <= 0.5) return fail(LTK_ERR_CONFIG, "tau must be > 0.5");
    if (p->mode != LTK_MODE_EXACT && p->mode != LTK_MODE_FAST)
        return fail(LTK_ERR_CONFIG, "unknown mode %d", p->mode);
    if (p->physics < 0 || p->physics > 2) return fail(LTK_ERR_CONFIG, "unknown physics");
    ltk_fluid *e = new (std::nothrow) ltk_fluid();
    if (!e) return fail(LTK_ERR_ALLOC, "host allocation failed");
    e->nx = nx;
    e->ny = ny;
    e->nzg = nz_global;
    e->nzl = nz_global / nranks;
    e->z0 = (long long)rank * e->nzl;
    e->rank = rank;
    e->nranks = nranks;
    e->vvl = vvl;
    e->prm = *p;
    e->slab.nx = nx;
    e->slab.ny = ny;
    e->slab.nzl = e->nzl;
    // component stride: whole planes, rounded up to 64 doubles (512 B)
    const long long raw = (e->nzl + 2) * nx * ny;
    e->slab.cstride = (raw + 63) / 64 * 64;
    int rc = check_slab(&e->slab, vvl);
    if (!rc && vvl > 2) rc = fail(LTK_ERR_PLAN, "engine vvl must be 1 or 2");
    if (rc) {
        delete e;
        return rc;
    }
    cudaGetDevice(&e->dev);
    const size_t dist_bytes = (size_t)e->slab.cstride * Q * sizeof(double);
    const size_t plane_bytes = (size_t)raw * sizeof(double);
    void *ptr = nullptr;
    for (int s = 0; s < 2; ++s)
        for (int d = 0; d < 2; ++d) {
            rc = ltk_malloc(&ptr, dist_bytes);
            if (rc) {
                ltk_fluid_destroy(e);
                return rc;
            }
            e->fg[s][d] = (double *)ptr;
        }
    e->phi_stride = (raw + 63) / 64 * 64;
    if ((rc = ltk_malloc(&ptr, 2 * (size_t)e->phi_stride * sizeof(double)))) {
        ltk_fluid_destroy(e);
        return rc;
    }
    e->phi = (double *)ptr;
    if ((rc = ltk_malloc(&ptr, (size_t)(e->nzl + 1) * sizeof(unsigned long long)))) {  // zeroed
        ltk_fluid_destroy(e);
        return rc;
    }
    e->fsync = (unsigned long long *)ptr;
    // row-blocked f/g by default (measured faster, bitwise identical: DESIGN.md §4);
    // SoA for odd nx (16-byte rows) or LTK_LAYOUT=0
    e->lay = nx % 2 == 0 ? row_lay(&e->slab) : soa_lay(&e->slab);
    if (const char *v = getenv("LTK_LAYOUT"))
        if (atoi(v) == LTK_LAYOUT_SOA) e->lay = soa_lay(&e->slab);
    if (const char *v = getenv("LTK_FUSE")) e->fuse = atoi(v) != 0;  // default off
    if (const char *v = getenv("LTK_PEER_OVERLAP")) e->peer_overlap = atoi(v) != 0;
    if (const char *v = getenv("LTK_FUSE_LAG")) e->fuse_lag = std::max(0, atoi(v));
    // mu followed by the stress form's 4 aux arrays (p_iso, grad phi), one
    // allocation so one IPC handle maps all of them
    if ((rc = ltk_malloc(&ptr, 5 * (size_t)e->phi_stride * sizeof(double)))) {
        ltk_fluid_destroy(e);
        return rc;
    }
    e->mu = (double *)ptr;
    if (cudaStreamCreateWithFlags(&e->st, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&e->comm_st, cudaStreamNonBlocking) != cudaSuccess) {
        ltk_fluid_destroy(e);
        return fail(LTK_ERR_DEVICE, "stream creation failed");
    }
    for (int k = 0; k < 3; ++k) {
        cudaEventCreateWithFlags(&e->ev_fork[k], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&e->ev_join[k], cudaEventDisableTiming);
    }
    if (!singular_word()) {
        ltk_fluid_destroy(e);
        return fail(LTK_ERR_DEVICE, "device error word unavailable");
    }
    if ((rc = ltk_malloc(&ptr, 2 * sizeof(unsigned long long)))) {
        ltk_fluid_destroy(e);
        return rc;
    }
    e->inbox = (unsigned long long *)ptr;
    if ((rc = ltk_malloc(&ptr, sizeof(int)))) {
        ltk_fluid_destroy(e);
        return rc;
    }
    e->peer_timeout = (int *)ptr;
    *out = e;
    return LTK_OK;
}

int ltk_fluid_destroy(ltk_fluid *e) {
    if (!e) return LTK_OK;
    if (e->st) cudaStreamSynchronize(e->st);
    if (e->comm_st) cudaStreamSynchronize(e->comm_st);
    drop_graphs(e);
    if (e->comm && nccl().ok) nccl().CommDestroy(e->comm);
    for (void *p : e->ipc_opened) cudaIpcCloseMemHandle(p);
    if (e->inbox) cudaFree(e->inbox);
    if (e->peer_timeout) cudaFree(e->peer_timeout);
    for (auto &s : e->fg)
        for (auto &p : s)
            if (p) cudaFree(p);
    if (e->phi) cudaFree(e->phi);
    if (e->fsync) cudaFree(e->fsync);
    if (e->mu) cudaFree(e->mu);
    for (int k = 0; k < 3; ++k) {
        if (e->ev_fork[k]) cudaEventDestroy(e->ev_fork[k]);
        if (e->ev_join[k]) cudaEventDestroy(e->ev_join[k]);
    }
    for (auto ev : e->ppool) cudaEventDestroy(ev);
    if (e->st) cudaStreamDestroy(e->st);
    if (e->comm_st) cudaStreamDestroy(e->comm_st);
    delete e;
    return LTK_OK;
}

int ltk_fluid_slab(const ltk_fluid *e, ltk_slab *s, int64_t *z0) {
    *s = e->slab;
    if (z0) *z0 = e->z0;
    return LTK_OK;
}

int ltk_fluid_buffers(const ltk_fluid *e, double **f, double **g, double **phi, double **mu) {
    if (f) *f = e->fg[e->cur][0];
    if (g) *g = e->fg[e->cur][1];
    // phi of the last step's input state (this state's before any step)
    if (phi) *phi = e->phi_of(e->step > 0 ? 1 - e->cur : e->cur);
    if (mu) *mu = e->mu;
    return LTK_OK;
}

int ltk_fluid_stream(const ltk_fluid *e, void **stream) {
    *stream = e->st;
    return LTK_OK;
}

int ltk_fluid_set_params(ltk_fluid *e, const ltk_fluid_params *p) {
    if (p->tau_f <= 0.5 || p->tau_g <= 0.5) return fail(LTK_ERR_CONFIG, "tau must be > 0.5");
    if (p->mode != LTK_MODE_EXACT && p->mode != LTK_MODE_FAST)
        return fail(LTK_ERR_CONFIG, "unknown mode %d", p->mode);
    if (p->physics < 0 || p->physics > 2) return fail(LTK_ERR_CONFIG, "unknown physics");
    e->prm = *p;
    drop_graphs(e);
    return LTK_OK;
}

int ltk_fluid_load(ltk_fluid *e, const double *f_src, const double *g_src, int64_t padded,
                   int64_t nz_src, int64_t z_src0, void *stream) {
    cudaStream_t st = stream ? as_stream(stream) : e->st;
    if (e->transport == kPeer) LTK_RC(peer_before_load(e, st));
    e->cur = 0;
    e->phi_lo = e->phi_hi = 0;  // phi of the loaded state not formed yet
    LTK_RC(transpose(&e->slab, e->lay, e->fg[0][0], const_cast<double *>(f_src), padded, nz_src,
                     z_src0, Q, true, st));
    LTK_RC(transpose(&e->slab, e->lay, e->fg[0][1], const_cast<double *>(g_src), padded, nz_src,
                     z_src0, Q, true, st));
    if (e->transport == kLocal) LTK_RC(wrap_state_halos(e, 0, 1, st));
    if (e->transport == kPeer) LTK_RC(peer_prime(e, 0, st));
    return LTK_OK;
}

int ltk_fluid_store(ltk_fluid *e, double *f_dst, double *g_dst, int64_t padded, int64_t nz_src,
                    int64_t z_src0, void *stream) {
    cudaStream_t st = stream ? as_stream(stream) : e->st;
    LTK_RC(transpose(&e->slab, e->lay, e->fg[e->cur][0], f_dst, padded, nz_src, z_src0, Q, false,
                     st));
    LTK_RC(transpose(&e->slab, e->lay, e->fg[e->cur][1], g_dst, padded, nz_src, z_src0, Q, false,
                     st));
    return LTK_OK;
}

int ltk_fluid_totals(ltk_fluid *e, double *out5) {
    double *partial = nullptr;
    LTK_CUDA(cudaMallocAsync(&partial, sizeof(double) * 5 * kTotBlocks, e->st));
    k_totals<<<kTotBlocks, kTotThreads, 0, e->st>>>(e->fg[e->cur][0], e->fg[e->cur][1], e->nx,
                                                   e->ny, e->nzl, e->lay.SI, e->lay.SZ,
                                                   e->lay.SY, partial);
    LTK_CHECK_LAUNCH("k_totals");
    std::vector<double> h(5 * kTotBlocks);
    LTK_CUDA(cudaMemcpyAsync(h.data(), partial, sizeof(double) * h.size(),
                             cudaMemcpyDeviceToHost, e->st));
    LTK_CUDA(cudaFreeAsync(partial, e->st));
    LTK_CUDA(cudaStreamSynchronize(e->st));
    for (int k = 0; k < 5; ++k) out5[k] = 0.0;
    for (int b = 0; b < kTotBlocks; ++b)
        for (int k = 0; k < 5; ++k) out5[k] += h[b * 5 + k];
    return LTK_OK;
}

int ltk_fluid_use_graph(ltk_fluid *e, int32_t enable) {
    drop_graphs(e);
    e->use_graph = enable != 0;
    return LTK_OK;
}

// Profiling: every profiled step records 4 events (start, after phi, after
// mu + halo, after collide-stream) on the engine stream; nothing waits on
// them until the window is read, so the timed stream runs undisturbed.
int ltk_fluid_profile(ltk_fluid *e, int32_t enable, float *ms4) {
    float acc[4] = {0, 0, 0, 0};
    if (!e->ppool.empty()) {
        LTK_CUDA(cudaEventSynchronize(e->ppool.back()));
        for (size_t k = 0; k + 3 < e->ppool.size(); k += 4) {
            float ms;
            cudaEventElapsedTime(&ms, e->ppool[k], e->ppool[k + 1]);
            acc[0] += ms;
            cudaEventElapsedTime(&ms, e->ppool[k + 1], e->ppool[k + 2]);
            acc[1] += ms;
            cudaEventElapsedTime(&ms, e->ppool[k + 2], e->ppool[k + 3]);
            acc[2] += ms;
            cudaEventElapsedTime(&ms, e->ppool[k], e->ppool[k + 3]);
            acc[3] += ms;
        }
        for (auto ev : e->ppool) cudaEventDestroy(ev);
        e->ppool.clear();
    }
    if (ms4)
        for (int k = 0; k < 4; ++k) ms4[k] = acc[k];
    e->prof = enable != 0;
    e->prof_steps = 0;
    return LTK_OK;
}

int ltk_fluid_run(ltk_fluid *e, int64_t nsteps, void *stream) {
    cudaStream_t st = stream ? as_stream(stream) : e->st;
    for (int64_t k = 0; k < nsteps; ++k) {
        const int s = e->cur;
        int nxt[2] = {0, 0};
        if (e->prof) {
            for (int k = 0; k < 4; ++k) {
                cudaEvent_t ev;
                LTK_CUDA(cudaEventCreate(&ev));
                e->ppool.push_back(ev);
                e->pev[k] = ev;
            }
            LTK_RC(enqueue_step(e, s, st, true, nxt));
            ++e->prof_steps;
        } else if (e->use_graph && e->transport == kLocal) {
            // one graph per (input state, whether its phi interior is formed)
            const int key = s + (e->phi_hi > e->phi_lo ? 2 : 0);
            if (!e->gexec[key]) {
                cudaGraph_t g;
                LTK_CUDA(cudaStreamBeginCapture(e->st, cudaStreamCaptureModeThreadLocal));
                int rc = enqueue_step(e, s, e->st, false, nxt);
                cudaError_t ce = cudaStreamEndCapture(e->st, &g);
                if (rc) return rc;
                if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture");
                ce = cudaGraphInstantiate(&e->gexec[key], g, 0);
                cudaGraphDestroy(g);
                if (ce != cudaSuccess) return cuda_fail(ce, "cudaGraphInstantiate");
                e->gnxt[key][0] = nxt[0];
                e->gnxt[key][1] = nxt[1];
            }
            nxt[0] = e->gnxt[key][0];
            nxt[1] = e->gnxt[key][1];
            LTK_CUDA(cudaGraphLaunch(e->gexec[key], st));
            count_launch(3);
        } else {
            LTK_RC(enqueue_step(e, s, st, false, nxt));
        }
        e->phi_lo = nxt[0];
        e->phi_hi = nxt[1];
        e->cur = 1 - s;
        ++e->step;
    }
    return LTK_OK;
}

// Fused collide-stream + next-state phi on/off and its lag (planes of slack
// between the collision front and the phi front).
int ltk_fluid_set_fuse(ltk_fluid *e, int32_t enable, int32_t extra_lag) {
    if (extra_lag < 0) return fail(LTK_ERR_CONFIG, "lag must be >= 0");
    e->fuse = enable != 0;
    e->fuse_lag = extra_lag;
    drop_graphs(e);
    return LTK_OK;
}

// ---- peer transport (CUDA IPC) ----
// An IPC handle names the whole driver allocation that contains a pointer
// (small cudaMalloc blocks share one), and the importer gets that
// allocation's base back; so the blob also carries each buffer's offset from
// its base (cuMemGetAddressRange, reached through the runtime's driver entry
// point), and identical handles are opened only once.
struct IpcBlob {
    cudaIpcMemHandle_t h[7];  // f0 g0 f1 g1 phi mu inbox
    unsigned long long off[7];
    long long SY;  // f/g layout (row stride) of the exporting slab
};
static_assert(sizeof(IpcBlob) <= LTK_IPC_BLOB_BYTES, "IPC blob too large");

typedef CUresult (*PfnGetAddressRange)(CUdeviceptr *, size_t *, CUdeviceptr);

static int alloc_base(void *p, unsigned long long *off) {
    static PfnGetAddressRange fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *sym = nullptr;
        LTK_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &sym, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !sym)
            return fail(LTK_ERR_DEVICE, "cuMemGetAddressRange unavailable");
        fn = (PfnGetAddressRange)sym;
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (fn(&base, &size, (CUdeviceptr)p) != CUDA_SUCCESS)
        return fail(LTK_ERR_DEVICE, "cuMemGetAddressRange failed");
    *off = (unsigned long long)((CUdeviceptr)p - base);
    return LTK_OK;
}

int ltk_fluid_ipc_blob(ltk_fluid *e, char *blob) {
    IpcBlob b;
    void *ptrs[7] = {e->fg[0][0], e->fg[0][1], e->fg[1][0], e->fg[1][1], e->phi, e->mu,
                     e->inbox};
    for (int k = 0; k < 7; ++k) {
        LTK_CUDA(cudaIpcGetMemHandle(&b.h[k], ptrs[k]));
        LTK_RC(alloc_base(ptrs[k], &b.off[k]));
    }
    b.SY = e->lay.SY;
    memset(blob, 0, LTK_IPC_BLOB_BYTES);
    memcpy(blob, &b, sizeof b);
    return LTK_OK;
}

static int open_peer(ltk_fluid *e, const char *blob, ltk_fluid::Peer &p) {
    IpcBlob b;
    memcpy(&b, blob, sizeof b);
    if (b.SY != e->lay.SY) return fail(LTK_ERR_SHAPE, "peer slabs differ in layout");
    char *ptrs[7];
    for (int k = 0; k < 7; ++k) {
        void *base = nullptr;
        for (int j = 0; j < k; ++j)  // same allocation as an earlier buffer
            if (memcmp(&b.h[j], &b.h[k], sizeof(cudaIpcMemHandle_t)) == 0)
                base = ptrs[j] - b.off[j];
        if (!base) {
            cudaError_t ce = cudaIpcOpenMemHandle(&base, b.h[k], cudaIpcMemLazyEnablePeerAccess);
            if (ce != cudaSuccess) return cuda_fail(ce, "cudaIpcOpenMemHandle");
            e->ipc_opened.push_back(base);
        }
        ptrs[k] = (char *)base + b.off[k];
    }
    p.fg[0][0] = (double *)ptrs[0];
    p.fg[0][1] = (double *)ptrs[1];
    p.fg[1][0] = (double *)ptrs[2];
    p.fg[1][1] = (double *)ptrs[3];
    p.phi[0] = (double *)ptrs[4];
    p.phi[1] = p.phi[0] + e->phi_stride;  // same layout on every slab
    p.mu = (double *)ptrs[5];
    p.inbox = (unsigned long long *)ptrs[6];
    return LTK_OK;
}

int ltk_fluid_attach_peers(ltk_fluid *e, const char *up_blob, const char *dn_blob) {
    if (e->nranks < 2) return fail(LTK_ERR_CONFIG, "peer transport needs >= 2 slabs");
    if (e->transport != kLocal) return fail(LTK_ERR_CONFIG, "transport already attached");
    LTK_RC(preload_step_kernels());
    preload_cs_tma((int)e->nx);
    LTK_RC(open_peer(e, up_blob, e->up));
    if (memcmp(up_blob, dn_blob, sizeof(IpcBlob)) == 0)
        e->dn = e->up;  // two slabs: both neighbours are the same rank
    else
        LTK_RC(open_peer(e, dn_blob, e->dn));
    // complete before returning: the legacy-stream memset must not land after
    // a neighbour's first progress signal (the caller barriers after attach)
    LTK_CUDA(cudaMemset(e->inbox, 0, 2 * sizeof(unsigned long long)));
    LTK_CUDA(cudaMemset(e->peer_timeout, 0, sizeof(int)));
    LTK_CUDA(cudaStreamSynchronize(0));
    e->transport = kPeer;
    drop_graphs(e);
    return LTK_OK;
}

static void peer_from_engine(ltk_fluid::Peer &p, const ltk_fluid *o) {
    for (int st = 0; st < 2; ++st)
        for (int d = 0; d < 2; ++d) p.fg[st][d] = o->fg[st][d];
    p.phi[0] = o->phi_of(0);
    p.phi[1] = o->phi_of(1);
    p.mu = o->mu;
    p.inbox = o->inbox;
}

int ltk_fluid_attach_peer_engines(ltk_fluid *e, const ltk_fluid *up, const ltk_fluid *dn) {
    if (e->nranks < 2) return fail(LTK_ERR_CONFIG, "peer transport needs >= 2 slabs");
    if (e->transport != kLocal) return fail(LTK_ERR_CONFIG, "transport already attached");
    if (up->slab.cstride != e->slab.cstride || dn->slab.cstride != e->slab.cstride ||
        up->lay.SY != e->lay.SY || dn->lay.SY != e->lay.SY)
        return fail(LTK_ERR_SHAPE, "peer slabs differ in layout");
    LTK_RC(preload_step_kernels());
    preload_cs_tma((int)e->nx);
    peer_from_engine(e->up, up);
    peer_from_engine(e->dn, dn);
    // complete before returning: the legacy-stream memset must not land after
    // a neighbour's first progress signal (the caller barriers after attach)
    LTK_CUDA(cudaMemset(e->inbox, 0, 2 * sizeof(unsigned long long)));
    LTK_CUDA(cudaMemset(e->peer_timeout, 0, sizeof(int)));
    LTK_CUDA(cudaStreamSynchronize(0));
    e->transport = kPeer;
    drop_graphs(e);
    return LTK_OK;
}

int ltk_fluid_peer_timeout(ltk_fluid *e, int32_t *timed_out) {
    LTK_CUDA(cudaStreamSynchronize(e->st));
    int v = 0;
    LTK_CUDA(cudaMemcpy(&v, e->peer_timeout, sizeof v, cudaMemcpyDeviceToHost));
    *timed_out = v;
    return LTK_OK;
}

int ltk_fluid_cs_variant(int32_t variant, int32_t *previous) {
    if (previous) *previous = cs_variant();
    if (variant >= 0) {
        if (variant != LTK_CS_REG && variant != LTK_CS_TMA)
            return fail(LTK_ERR_CONFIG, "unknown collide-stream variant %d", variant);
        cs_variant() = variant;
    }
    return LTK_OK;
}

int ltk_fluid_mu_variant(int32_t variant, int32_t *previous) {
    if (previous) *previous = mu_variant();
    if (variant >= 0) {
        if (variant > LTK_MU_BLK) return fail(LTK_ERR_CONFIG, "unknown mu variant %d", variant);
        mu_variant() = variant;
    }
    return LTK_OK;
}

int ltk_nccl_available(void) { return nccl().ok ? 1 : 0; }

int ltk_nccl_unique_id(char id[128]) {
    if (!nccl().ok) return fail(LTK_ERR_DEVICE, "libnccl.so.2 not loadable");
    ncclUniqueId u;
    LTK_NCCL(nccl().GetUniqueId(&u));
    memcpy(id, u.internal, 128);
    return LTK_OK;
}

int ltk_fluid_attach_nccl(ltk_fluid *e, const char id[128]) {
    if (!nccl().ok) return fail(LTK_ERR_DEVICE, "libnccl.so.2 not loadable");
    if (!is_soa(e->lay, &e->slab)) {  // NCCL sends contiguous SoA component planes
        e->lay = soa_lay(&e->slab);
        e->cur = 0;
        e->phi_lo = e->phi_hi = 0;
    }
    ncclUniqueId u;
    memcpy(u.internal, id, 128);
    LTK_NCCL(nccl().CommInitRank(&e->comm, e->nranks, u, e->rank));
    e->transport = kNccl;
    drop_graphs(e);
    return LTK_OK;
}

}  // extern "C"

extern "C" int ltk_fluid_set_layout(ltk_fluid *e, int32_t layout, int32_t *previous) {
    if (previous) *previous = is_soa(e->lay, &e->slab) ? LTK_LAYOUT_SOA : LTK_LAYOUT_ROW;
    if (layout < 0) return LTK_OK;  // query
    if (layout != LTK_LAYOUT_SOA && layout != LTK_LAYOUT_ROW)
        return fail(LTK_ERR_CONFIG, "unknown layout %d", layout);
    if (e->transport != kLocal)
        return fail(LTK_ERR_CONFIG, "set the layout before attaching a transport");
    if (layout == LTK_LAYOUT_ROW && e->nx % 2)
        return fail(LTK_ERR_SHAPE, "the row-blocked layout needs an even nx");
    e->lay = layout == LTK_LAYOUT_ROW ? row_lay(&e->slab) : soa_lay(&e->slab);
    e->cur = 0;
    e->phi_lo = e->phi_hi = 0;
    drop_graphs(e);
    return LTK_OK;
}
