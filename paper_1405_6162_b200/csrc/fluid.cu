// fluid.cu -- the full D3Q19 binary-fluid timestep on B200: C-ABI launchers
// of the kernels in fluid_kernels.cuh, host-order <-> slab transposes, halo
// faces, and the C++ step engine (one slab with a periodic z wrap, or z-slabs
// joined by peer stores over NVLink or by NCCL, halos overlapped with the
// interior planes).
//
// No reference counterpart (reference pkg/README.md:34-35: collision only);
// specification in DESIGN.md §2-§5.  The collision arithmetic is the
// reference's (kernels.py:89-125) with the free-energy force terms added.
#include <cuda.h>  // CUresult / CUdeviceptr for the driver entry point (no libcuda link)
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl.so.2 is dlopen'ed at run time

#include <algorithm>
#include <cstring>
#include <new>
#include <vector>

#include "fluid_kernels.cuh"

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
    if ((long long)s->nx * s->ny * (s->nzl + 4) >= (1LL << 31))
        return fail(LTK_ERR_SHAPE, "slab too large for 32-bit thread indexing");
    return LTK_OK;
}

static void fill_args(FluidArgs &a, const ltk_slab *s, const ltk_fluid_params *p) {
    memset(&a, 0, sizeof a);
    a.nx = (int)s->nx;
    a.ny = (int)s->ny;
    a.nzl = (int)s->nzl;
    a.PL = s->nx * s->ny;
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

static int check_params(const ltk_fluid_params *p) {
    if (!p) return fail(LTK_ERR_CONFIG, "null params");
    if (p->tau_f <= 0.5 || p->tau_g <= 0.5) return fail(LTK_ERR_CONFIG, "tau must be > 0.5");
    if (p->mode != LTK_MODE_EXACT && p->mode != LTK_MODE_FAST)
        return fail(LTK_ERR_CONFIG, "unknown mode %d", p->mode);
    if (p->physics < 0 || p->physics > 2) return fail(LTK_ERR_CONFIG, "unknown physics %d", p->physics);
    return LTK_OK;
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

// mu stencil kernel (process-wide): LTK_MU_AUTO = the shared-memory tile
// kernel where the shape allows it, else the plain one; LTK_MU_PLAIN = plain.
static int &mu_variant() {
    static int v = LTK_MU_AUTO;
    return v;
}

static int launch_mu(const FluidArgs &a, int vvl, cudaStream_t st) {
    if (a.nthreads <= 0) return LTK_OK;
    if (mu_variant() == LTK_MU_AUTO && mu_tile_ok(a.nx, a.ny)) {
        dim3 grid((unsigned)(a.nx / 32), (unsigned)(a.ny / 8),
                  (unsigned)((a.nplanes + kMuTileZ - 1) / kMuTileZ));
        k_mu_tile<kMuTileZ><<<grid, dim3(32, 8), 0, st>>>(a);
        LTK_CHECK_LAUNCH("k_mu_tile");
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

template <int MODE, int PHYS, int T1>
static void launch_cs_t(const FluidArgs &a, int vvl, cudaStream_t st) {
    const unsigned g = grid_for(a.nthreads, kTPB);
    if (vvl == 2)
        k_collide_stream<2, MODE, PHYS, T1><<<g, kTPB, 0, st>>>(a);
    else
        k_collide_stream<1, MODE, PHYS, T1><<<g, kTPB, 0, st>>>(a);
}

template <int PHYS>
static void launch_cs_p(const FluidArgs &a, int vvl, int mode, cudaStream_t st) {
    if (mode != LTK_MODE_EXACT) return launch_cs_t<LTK_MODE_FAST, PHYS, 0>(a, vvl, st);
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
    if (vvl > 2) return fail(LTK_ERR_PLAN, "collide-stream supports vvl 1 and 2");
    if (phys == 0) launch_cs_p<0>(a, vvl, mode, st);
    else if (phys == 1) launch_cs_p<1>(a, vvl, mode, st);
    else launch_cs_p<2>(a, vvl, mode, st);
    LTK_CHECK_LAUNCH("k_collide_stream");
    return LTK_OK;
}

// ------------------------------------------------------------------ plane copies
// Each copy moves `rows` rows of `row` doubles (row even); rows are sstride
// doubles apart in the source and dstride apart in the destination.
struct PlaneCopies {
    const double *src[24];
    double *dst[24];
    int n;
    long long rows, row, sstride, dstride;
};

__global__ void __launch_bounds__(256) k_plane_copy(const PlaneCopies pc) {
    const int j = blockIdx.y;
    const double *s = pc.src[j];
    double *d = pc.dst[j];
    const long long r2 = pc.row / 2, n2 = pc.rows * r2;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / r2, c = 2 * (i - r * r2);
        *reinterpret_cast<double2 *>(d + r * pc.dstride + c) =
            *reinterpret_cast<const double2 *>(s + r * pc.sstride + c);
    }
}

static int run_plane_copies(const PlaneCopies &pc, cudaStream_t st) {
    if (pc.n == 0) return LTK_OK;
    dim3 grid((unsigned)std::min<long long>((pc.rows * pc.row / 2 + 255) / 256, 148 * 4), pc.n);
    k_plane_copy<<<grid, 256, 0, st>>>(pc);
    LTK_CHECK_LAUNCH("k_plane_copy");
    return LTK_OK;
}

constexpr int kUp[5] = {5, 11, 13, 15, 17};    // cz = +1
constexpr int kDown[5] = {6, 12, 14, 16, 18};  // cz = -1

// f/g storage layout: element (comp i, storage plane zs, row y, x) at
// i*SI + zs*SZ + y*SY + x.  SoA (component-major planes) is the C-ABI slab
// layout; the engine holds its state row-blocked by default (the 19
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

// A set of copies of component planes of layout L (src side, dst side).
static PlaneCopies plane_copies(const Lay &Ls, const Lay &Ld, const ltk_slab *s) {
    PlaneCopies pc;
    memset(&pc, 0, sizeof pc);
    const bool cs = Ls.SY == s->nx, cd = Ld.SY == s->nx;  // plane contiguous?
    if (cs && cd) {
        pc.rows = 1;
        pc.row = s->nx * s->ny;
    } else {
        pc.rows = s->ny;
        pc.row = s->nx;
    }
    pc.sstride = Ls.SY;
    pc.dstride = Ld.SY;
    return pc;
}

// The contiguous "face" layout of packed component planes: plane k at k*PL.
static inline Lay face_lay(const ltk_slab *s) { return {s->nx * s->ny, 0, s->nx}; }

// ------------------------------------------------------------------ transposes
// host order site (x*ny + y)*nzg + z  <->  slab (z - z0 + 1)*SZ + y*SY + x.
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
    dim3 block(32, 8);
    dim3 grid((unsigned)((s->nx + 31) / 32), (unsigned)((s->nzl + 31) / 32),
              (unsigned)(s->ny * ncomp));
    if ((long long)s->ny * ncomp > 65535) return fail(LTK_ERR_SHAPE, "ny*ncomp exceeds 65535");
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
    ltk::Lay lay{};  // f/g layout (row-blocked by default for even nx)
    double *fg[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [state][f/g]
    // phi: nzl + 2 planes; mu: nzl + 4 planes followed by the stress form's
    // 4 aux arrays in mu's layout (one allocation, so one IPC handle maps all)
    double *phi = nullptr, *mu = nullptr;
    long long mu_stride = 0;
    // error words of this engine: [0] singular site, [1] peer wait timeout
    long long *err = nullptr;
    bool failed = false;  // a peer wait timed out: the state is not trustworthy
    int cur = 0;
    bool peer_overlap = true;  // peer transport: boundary planes on comm_st (env LTK_PEER_OVERLAP)
    cudaStream_t st = nullptr, comm_st = nullptr;
    cudaEvent_t ev_fork[3] = {}, ev_join[3] = {};
    ncclComm_t comm = nullptr;
    double *face = nullptr;  // NCCL: send up, send down, recv from below, recv from above (10 planes each)
    // transport between slabs: LOCAL (one slab, periodic images into itself),
    // NCCL (face exchanges on comm_st), PEER (CUDA IPC: halo images stored by
    // the kernels straight into the neighbours' buffers over NVLink)
    int transport = 0;
    struct Peer {
        double *fg[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
        double *phi = nullptr, *mu = nullptr;
        unsigned long long *inbox = nullptr;
    } up, dn;
    unsigned long long *inbox = nullptr;  // [2]: progress of the slab below / above
    std::vector<void *> ipc_opened;
    long long step = 0;   // timesteps taken (lockstep across slabs)
    bool primed = false;  // peer transport: halos re-primed by a load since the last step
    bool use_graph = false;
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};  // [input state]
    bool prof = false;
    cudaEvent_t pev[4] = {};          // events of the step being enqueued
    std::vector<cudaEvent_t> ppool;   // 4 per profiled step, read at the end
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
    a.phi = a.phi_out = e->phi;
    a.mu = a.mu_out = e->mu;
    a.astride = e->mu_stride;
    a.aux = e->prm.physics == 2 ? e->mu + e->mu_stride : nullptr;
    a.err = e->err;
    if (e->transport == kLocal) {  // periodic images into this slab
        a.wrap_local = 1;
        a.img_f_up = a.img_f_dn = a.f_out;
        a.img_g_up = a.img_g_dn = a.g_out;
        a.img_phi_up = a.img_phi_dn = e->phi;
        a.img_mu_up = a.img_mu_dn = e->mu;
    } else if (e->transport == kPeer) {  // images into the neighbours over NVLink
        a.img_f_up = e->up.fg[1 - in_state][0];
        a.img_g_up = e->up.fg[1 - in_state][1];
        a.img_f_dn = e->dn.fg[1 - in_state][0];
        a.img_g_dn = e->dn.fg[1 - in_state][1];
        a.img_phi_up = e->up.phi;
        a.img_phi_dn = e->dn.phi;
        a.img_mu_up = e->up.mu;
        a.img_mu_dn = e->dn.mu;
    }
    return a;
}

#define LTK_RC(x)              \
    do {                       \
        int rc_ = (x);         \
        if (rc_) return rc_;   \
    } while (0)

// One NCCL halo exchange group on comm_st.  kind 0: the f/g components of
// state `s` that cross the faces, packed into one contiguous 10-plane face
// per direction (any f/g layout) and unpacked into the halo planes; kind 1:
// phi (one plane per face); kind 2: mu (two planes per face) and, for the
// stress form, its 4 aux arrays.  Send order per peer is fixed (up, then
// down) and receives mirror it, which keeps the matching right even when
// both neighbours are the same rank (P = 2) or this rank itself (P = 1).
static int exchange(ltk_fluid *e, int kind, int s) {
    Nccl &n = nccl();
    const int up = (e->rank + 1) % e->nranks, down = (e->rank + e->nranks - 1) % e->nranks;
    const long long PL = e->nx * e->ny, nzl = e->nzl;
    const ltk_slab *sl = &e->slab;
    cudaStream_t cs = e->comm_st;
    if (kind == 0) {
        const long long F = 10 * PL;
        double *s_up = e->face, *s_dn = e->face + F, *r_lo = e->face + 2 * F, *r_hi = e->face + 3 * F;
        PlaneCopies pc = plane_copies(e->lay, face_lay(sl), sl);
        for (int d = 0; d < 2; ++d)
            for (int j = 0; j < 5; ++j) {
                pc.src[pc.n] = plane(e->fg[s][d], e->lay, kUp[j], nzl);
                pc.dst[pc.n] = s_up + (long long)(5 * d + j) * PL;
                ++pc.n;
                pc.src[pc.n] = plane(e->fg[s][d], e->lay, kDown[j], 1);
                pc.dst[pc.n] = s_dn + (long long)(5 * d + j) * PL;
                ++pc.n;
            }
        LTK_RC(run_plane_copies(pc, cs));
        LTK_NCCL(n.GroupStart());
        LTK_NCCL(n.Send(s_up, F, ncclFloat64, up, e->comm, cs));
        LTK_NCCL(n.Send(s_dn, F, ncclFloat64, down, e->comm, cs));
        LTK_NCCL(n.Recv(r_lo, F, ncclFloat64, down, e->comm, cs));
        LTK_NCCL(n.Recv(r_hi, F, ncclFloat64, up, e->comm, cs));
        LTK_NCCL(n.GroupEnd());
        PlaneCopies pu = plane_copies(face_lay(sl), e->lay, sl);
        for (int d = 0; d < 2; ++d)
            for (int j = 0; j < 5; ++j) {
                pu.src[pu.n] = r_lo + (long long)(5 * d + j) * PL;
                pu.dst[pu.n] = plane(e->fg[s][d], e->lay, kUp[j], 0);
                ++pu.n;
                pu.src[pu.n] = r_hi + (long long)(5 * d + j) * PL;
                pu.dst[pu.n] = plane(e->fg[s][d], e->lay, kDown[j], nzl + 1);
                ++pu.n;
            }
        return run_plane_copies(pu, cs);
    }
    LTK_NCCL(n.GroupStart());
    if (kind == 1) {  // phi: storage zs = z + 1
        double *b = e->phi;
        LTK_NCCL(n.Send(b + nzl * PL, PL, ncclFloat64, up, e->comm, cs));
        LTK_NCCL(n.Send(b + 1 * PL, PL, ncclFloat64, down, e->comm, cs));
        LTK_NCCL(n.Recv(b + 0 * PL, PL, ncclFloat64, down, e->comm, cs));
        LTK_NCCL(n.Recv(b + (nzl + 1) * PL, PL, ncclFloat64, up, e->comm, cs));
    } else {  // mu (+ aux): storage zs = z + 2, two planes per face
        const int nb = e->prm.physics == 2 ? 5 : 1;
        for (int k = 0; k < nb; ++k) {
            double *b = e->mu + (long long)k * e->mu_stride;
            LTK_NCCL(n.Send(b + nzl * PL, 2 * PL, ncclFloat64, up, e->comm, cs));  // z = nzl-2, nzl-1
            LTK_NCCL(n.Send(b + 2 * PL, 2 * PL, ncclFloat64, down, e->comm, cs));  // z = 0, 1
        }
        for (int k = 0; k < nb; ++k) {
            double *b = e->mu + (long long)k * e->mu_stride;
            LTK_NCCL(n.Recv(b, 2 * PL, ncclFloat64, down, e->comm, cs));                // z = -2, -1
            LTK_NCCL(n.Recv(b + (nzl + 2) * PL, 2 * PL, ncclFloat64, up, e->comm, cs));  // z = nzl, nzl+1
        }
    }
    LTK_NCCL(n.GroupEnd());
    return LTK_OK;
}

static int enqueue_step_peer(ltk_fluid *e, int s, cudaStream_t st);

// Plane ranges of the slab phases.  phi: the boundary planes
// 0, nzl-1 need the f/g halos.  mu: 0, nzl-1 need the phi halos.  collide-
// stream: planes 0, 1, nzl-2, nzl-1 need the mu halos (the force reads mu at
// z +- 2), 0 and nzl-1 also the f/g and phi halos; with physics 0 only the
// f/g halos matter, so the boundary is 0, nzl-1.
struct Ranges {
    long long lo0, lo1, hi0, hi1;  // boundary [lo0, lo1) and [hi0, hi1)
    long long in0, in1;            // interior
};
static Ranges ranges_of(long long nzl, int depth) {
    Ranges r;
    r.lo0 = 0;
    r.lo1 = std::min<long long>(depth, nzl);
    r.hi0 = std::max<long long>(r.lo1, nzl - depth);
    r.hi1 = nzl;
    r.in0 = r.lo1;
    r.in1 = r.hi0;
    return r;
}

// Enqueue one timestep reading state `s` and writing state 1 - s.
static int enqueue_step(ltk_fluid *e, int s, cudaStream_t st) {
    if (e->transport == kPeer) return enqueue_step_peer(e, s, st);
    FluidArgs a = engine_args(e, s);
    const int vvl = e->vvl, mode = e->prm.mode, phys = e->prm.physics;
    const long long nzl = e->nzl;
    const bool prof = e->prof;
    auto run = [&](long long lo, long long hi, auto launch_one) -> int {
        if (hi <= lo) return LTK_OK;
        set_planes(a, vvl, lo, hi);
        return launch_one();
    };
    auto phi_st = [&] { return launch_phi(a, vvl, st); };
    auto mu_st = [&] { return launch_mu(a, vvl, st); };
    auto cs_st = [&] { return launch_cs(a, vvl, mode, phys, st); };
    if (prof) cudaEventRecord(e->pev[0], st);
    if (e->transport == kLocal) {
        // single slab, periodic z: the kernels write the halo images themselves
        LTK_RC(run(0, nzl, phi_st));
        if (prof) cudaEventRecord(e->pev[1], st);
        if (phys >= 1) LTK_RC(run(0, nzl, mu_st));
        if (prof) cudaEventRecord(e->pev[2], st);
        LTK_RC(run(0, nzl, cs_st));
        if (prof) cudaEventRecord(e->pev[3], st);
        return LTK_OK;
    }
    // NCCL z-slabs: each exchange overlaps the interior planes of the next kernel
    auto fork_exchange = [&](int k, int kind) -> int {
        LTK_CUDA(cudaEventRecord(e->ev_fork[k], st));
        LTK_CUDA(cudaStreamWaitEvent(e->comm_st, e->ev_fork[k], 0));
        LTK_RC(exchange(e, kind, s));
        LTK_CUDA(cudaEventRecord(e->ev_join[k], e->comm_st));
        return LTK_OK;
    };
    auto join = [&](int k) -> int {
        LTK_CUDA(cudaStreamWaitEvent(st, e->ev_join[k], 0));
        return LTK_OK;
    };
    const Ranges r1 = ranges_of(nzl, 1), r2 = ranges_of(nzl, phys >= 1 ? 2 : 1);
    // (1) f/g faces || phi interior; then phi boundary
    LTK_RC(fork_exchange(0, 0));
    LTK_RC(run(r1.in0, r1.in1, phi_st));
    LTK_RC(join(0));
    LTK_RC(run(r1.lo0, r1.lo1, phi_st));
    LTK_RC(run(r1.hi0, r1.hi1, phi_st));
    if (prof) cudaEventRecord(e->pev[1], st);
    if (phys >= 1) {
        // (2) phi faces || mu interior; then mu boundary
        LTK_RC(fork_exchange(1, 1));
        LTK_RC(run(r1.in0, r1.in1, mu_st));
        LTK_RC(join(1));
        LTK_RC(run(r1.lo0, r1.lo1, mu_st));
        LTK_RC(run(r1.hi0, r1.hi1, mu_st));
        // (3) mu faces || collide-stream interior
        LTK_RC(fork_exchange(2, 2));
    }
    if (prof) cudaEventRecord(e->pev[2], st);
    LTK_RC(run(r2.in0, r2.in1, cs_st));
    if (phys >= 1) LTK_RC(join(2));
    LTK_RC(run(r2.lo0, r2.lo1, cs_st));
    LTK_RC(run(r2.hi0, r2.hi1, cs_st));
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

// Wait until both neighbours reached `target`.  Never hang the GPU: after
// ~8 s the wait records the timeout in the engine's error word [1] and
// returns; ltk_fluid_sync then reports LTK_ERR_DEVICE and the engine refuses
// further steps (its halos are stale).
__global__ void k_peer_wait(const unsigned long long *inbox, unsigned long long target,
                            long long *err) {
    long long spins = 0;
    while (ld_acquire_sys(inbox) < target || ld_acquire_sys(inbox + 1) < target) {
        if (++spins > (1LL << 25) || *(volatile long long *)(err + 1) != 0) {
            atomicExch(reinterpret_cast<unsigned long long *>(err + 1), 1ull);
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
    k_peer_wait<<<1, 1, 0, st>>>(e->inbox, target, e->err);
    LTK_CHECK_LAUNCH("k_peer_wait");
    return LTK_OK;
}

// One timestep with the peer transport.  Counter protocol per step t (each
// slab pushes its counter into the neighbours' inboxes; waits are ">="):
//   4t+1  f/g halo images of state t re-primed after a load (peer_prime)
//   4t+2  phi images sent      4t+3  mu images sent
//   4t+4  f/g images of state t+1 sent (= "state t+1 ready", 4(t+1))
// Boundary planes run on a second stream (bs): a phase's boundary planes need
// the neighbours' halos and the previous phase, never this phase's interior,
// so progress wait + boundary kernels (with their peer stores) + signal run
// concurrently with the interior kernel; the streams join before the next
// phase.  The mu phase signals after the join: its interior launch writes the
// images of planes 1 and nzl-2 too.  overlap off: everything in order on st.
static int enqueue_step_peer(ltk_fluid *e, int s, cudaStream_t st) {
    FluidArgs a = engine_args(e, s);
    const int vvl = e->vvl, mode = e->prm.mode, phys = e->prm.physics;
    const long long nzl = e->nzl;
    const bool prof = e->prof;
    const unsigned long long t4 = 4ULL * (unsigned long long)e->step;
    cudaStream_t bs = e->peer_overlap ? e->comm_st : st;
    auto run = [&](long long lo, long long hi, auto launch_one) -> int {
        if (hi <= lo) return LTK_OK;
        set_planes(a, vvl, lo, hi);
        return launch_one();
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
    auto cs_a = [&] { return launch_cs(a, vvl, mode, phys, st); };
    auto cs_b = [&] { return launch_cs(a, vvl, mode, phys, bs); };
    const Ranges r1 = ranges_of(nzl, 1), r2 = ranges_of(nzl, phys >= 1 ? 2 : 1);
    if (prof) cudaEventRecord(e->pev[0], st);
    // phi: interior || (f/g halos of state s -> boundary planes -> signal 4t+2)
    LTK_RC(fork(0));
    LTK_RC(peer_wait(e, t4 + (e->primed ? 1 : 0), bs));
    e->primed = false;
    LTK_RC(run(r1.lo0, r1.lo1, phi_b));
    LTK_RC(run(r1.hi0, r1.hi1, phi_b));
    LTK_RC(peer_signal(e, t4 + 2, bs));
    LTK_RC(run(r1.in0, r1.in1, phi_a));
    LTK_RC(join(0));
    if (prof) cudaEventRecord(e->pev[1], st);
    // mu: interior || (phi halos -> boundary planes); join; signal 4t+3
    if (phys >= 1) {
        LTK_RC(fork(1));
        LTK_RC(peer_wait(e, t4 + 2, bs));
        LTK_RC(run(r1.lo0, r1.lo1, mu_b));
        LTK_RC(run(r1.hi0, r1.hi1, mu_b));
        LTK_RC(run(r1.in0, r1.in1, mu_a));
        LTK_RC(join(1));
    }
    LTK_RC(peer_signal(e, t4 + 3, st));
    if (prof) cudaEventRecord(e->pev[2], st);
    // collide-stream: interior || (mu halos -> boundary planes -> signal 4t+4)
    LTK_RC(fork(2));
    LTK_RC(peer_wait(e, t4 + 3, bs));
    LTK_RC(run(r2.lo0, r2.lo1, cs_b));
    LTK_RC(run(r2.hi0, r2.hi1, cs_b));
    LTK_RC(peer_signal(e, t4 + 4, bs));
    LTK_RC(run(r2.in0, r2.in1, cs_a));
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
    PlaneCopies pc = plane_copies(e->lay, e->lay, &e->slab);
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
}

template <int PHYS>
static void preload_cs(cudaFuncAttributes &fa) {
    preload_cs_t<LTK_MODE_FAST, PHYS, 0>(fa);
    preload_cs_t<LTK_MODE_EXACT, PHYS, 0>(fa);
    preload_cs_t<LTK_MODE_EXACT, PHYS, 1>(fa);
    preload_cs_t<LTK_MODE_EXACT, PHYS, 2>(fa);
    preload_cs_t<LTK_MODE_EXACT, PHYS, 3>(fa);
}

static int preload_step_kernels() {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_phi<1>);
    cudaFuncGetAttributes(&fa, k_phi<2>);
    cudaFuncGetAttributes(&fa, k_phi<4>);
    cudaFuncGetAttributes(&fa, k_mu<1>);
    cudaFuncGetAttributes(&fa, k_mu<2>);
    cudaFuncGetAttributes(&fa, k_mu<4>);
    cudaFuncGetAttributes(&fa, k_mu_tile<kMuTileZ>);
    cudaFuncGetAttributes(&fa, k_plane_copy);
    cudaFuncGetAttributes(&fa, k_peer_wait);
    cudaFuncGetAttributes(&fa, k_peer_signal);
    cudaFuncGetAttributes(&fa, k_transpose<true>);
    cudaFuncGetAttributes(&fa, k_transpose<false>);
    cudaFuncGetAttributes(&fa, k_totals);
    preload_cs<0>(fa);
    preload_cs<1>(fa);
    preload_cs<2>(fa);
    LTK_CUDA(cudaGetLastError());
    return LTK_OK;
}

// Periodic z wrap of one slab's halos from its own owned planes.  which:
// bit 0 f/g crossing components (layout L), bit 1 phi (1 plane per face),
// bit 2 mu (2 planes per face, plane hz holds plane hz mod nzl).
static int wrap_halos(const ltk_slab *s, const Lay &L, double *f, double *g, double *phi,
                      double *mu, int which, cudaStream_t st) {
    const long long nzl = s->nzl, PL = s->nx * s->ny;
    if (which & 1) {
        PlaneCopies pc = plane_copies(L, L, s);
        for (int j = 0; j < 5; ++j)
            for (double *b : {f, g}) {
                pc.src[pc.n] = plane(b, L, kUp[j], nzl);
                pc.dst[pc.n++] = plane(b, L, kUp[j], 0);
                pc.src[pc.n] = plane(b, L, kDown[j], 1);
                pc.dst[pc.n++] = plane(b, L, kDown[j], nzl + 1);
            }
        LTK_RC(run_plane_copies(pc, st));
    }
    PlaneCopies pc;
    memset(&pc, 0, sizeof pc);
    pc.rows = 1;
    pc.row = PL;
    if ((which & 2) && phi) {
        pc.src[pc.n] = phi + nzl * PL;
        pc.dst[pc.n++] = phi;
        pc.src[pc.n] = phi + PL;
        pc.dst[pc.n++] = phi + (nzl + 1) * PL;
    }
    if ((which & 4) && mu) {
        for (long long hz : {-2LL, -1LL, nzl, nzl + 1}) {
            const long long src = ((hz % nzl) + nzl) % nzl;
            pc.src[pc.n] = mu + (src + 2) * PL;
            pc.dst[pc.n++] = mu + (hz + 2) * PL;
        }
    }
    return run_plane_copies(pc, st);
}

}  // namespace ltk

using namespace ltk;

// ---------------------------------------------------------------- slab-level C ABI

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
    LTK_RC(check_params(p));
    if (z_lo < 0 || z_hi > s->nzl || z_hi < z_lo) return fail(LTK_ERR_BOUNDS, "plane range");
    FluidArgs a;
    fill_args(a, s, p);
    a.phi = phi;
    a.mu_out = mu;
    set_planes(a, 1, z_lo, z_hi);
    return launch_mu(a, 1, as_stream(stream));
}

int ltk_fluid_collide_stream(const ltk_slab *s, const double *f_in, const double *g_in,
                             const double *phi, const double *mu, double *f_out, double *g_out,
                             const ltk_fluid_params *p, int64_t z_lo, int64_t z_hi, int32_t vvl,
                             void *stream) {
    LTK_RC(check_slab(s, vvl));
    LTK_RC(check_params(p));
    if (p->physics == 2)
        return fail(LTK_ERR_CONFIG, "the stress form (physics 2) runs in the engine only");
    if (z_lo < 0 || z_hi > s->nzl || z_hi < z_lo) return fail(LTK_ERR_BOUNDS, "plane range");
    FluidArgs a;
    fill_args(a, s, p);
    a.f_in = f_in;
    a.g_in = g_in;
    a.phi = phi;
    a.mu = mu;
    a.f_out = f_out;
    a.g_out = g_out;
    cudaStream_t st = as_stream(stream);
    a.err = stream_word(st);
    if (!a.err) return fail(LTK_ERR_DEVICE, "stream error word unavailable");
    set_planes(a, vvl, z_lo, z_hi);
    return launch_cs(a, vvl, p->mode, p->physics, st);
}

int ltk_fluid_wrap_halos(const ltk_slab *s, double *f, double *g, double *phi, double *mu,
                         int32_t which, void *stream) {
    LTK_RC(check_slab(s, 1));
    return wrap_halos(s, soa_lay(s), f, g, phi, mu, which, as_stream(stream));
}

static int face_copy(const ltk_slab *s, double *f, double *g, double *buf, int32_t dir,
                     bool pack, cudaStream_t st) {
    LTK_RC(check_slab(s, 1));
    if (dir != 1 && dir != -1) return fail(LTK_ERR_CONFIG, "dir must be +1 or -1");
    const Lay L = soa_lay(s), B = face_lay(s);
    PlaneCopies pc = plane_copies(L, B, s);
    const int *comps = dir > 0 ? kUp : kDown;
    const long long zs = pack ? (dir > 0 ? s->nzl : 1) : (dir > 0 ? 0 : s->nzl + 1);
    for (int d = 0; d < 2; ++d)
        for (int j = 0; j < 5; ++j) {
            double *pl = plane(d ? g : f, L, comps[j], zs);
            double *bf = buf + (long long)pc.n * s->nx * s->ny;
            pc.src[pc.n] = pack ? pl : bf;
            pc.dst[pc.n] = pack ? bf : pl;
            ++pc.n;
        }
    return run_plane_copies(pc, st);
}

int ltk_fluid_pack_face(const ltk_slab *s, const double *f, const double *g, double *buf,
                        int32_t dir, void *stream) {
    return face_copy(s, const_cast<double *>(f), const_cast<double *>(g), buf, dir, true,
                     as_stream(stream));
}

int ltk_fluid_unpack_face(const ltk_slab *s, double *f, double *g, const double *buf,
                          int32_t dir, void *stream) {
    return face_copy(s, f, g, const_cast<double *>(buf), dir, false, as_stream(stream));
}

int ltk_fluid_scatter(const ltk_slab *s, const double *host, int64_t padded, int64_t nz_global,
                      int64_t z0, int32_t ncomp, double *slab, void *stream) {
    LTK_RC(check_slab(s, 1));
    return transpose(s, soa_lay(s), slab, const_cast<double *>(host), padded, nz_global, z0,
                     ncomp, true, as_stream(stream));
}

int ltk_fluid_gather(const ltk_slab *s, const double *slab, int64_t padded, int64_t nz_global,
                     int64_t z0, int32_t ncomp, double *host, void *stream) {
    LTK_RC(check_slab(s, 1));
    return transpose(s, soa_lay(s), const_cast<double *>(slab), host, padded, nz_global, z0,
                     ncomp, false, as_stream(stream));
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

int ltk_fluid_mu_variant(int32_t variant, int32_t *previous) {
    if (previous) *previous = mu_variant();
    if (variant >= 0) {
        if (variant != LTK_MU_AUTO && variant != LTK_MU_PLAIN)
            return fail(LTK_ERR_CONFIG, "unknown mu variant %d", variant);
        mu_variant() = variant;
    }
    return LTK_OK;
}

// ---------------------------------------------------------------- engine API

int ltk_fluid_destroy(ltk_fluid *e);

static int engine_alloc(void **p, size_t bytes, ltk_fluid *e) {
    int rc = ltk_malloc(p, bytes);
    if (rc) ltk_fluid_destroy(e);
    return rc;
}

int ltk_fluid_create(int64_t nx, int64_t ny, int64_t nz_global, int32_t rank, int32_t nranks,
                     const ltk_fluid_params *p, int32_t vvl, ltk_fluid **out) {
    *out = nullptr;
    LTK_RC(check_params(p));
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(LTK_ERR_CONFIG, "bad rank/nranks");
    if (nz_global % nranks)
        return fail(LTK_ERR_SHAPE, "nz %lld not divisible by %d ranks", (long long)nz_global,
                    nranks);
    if (vvl != 1 && vvl != 2) return fail(LTK_ERR_PLAN, "engine vvl must be 1 or 2");
    if (nranks > 1 && nz_global / nranks < 2)
        return fail(LTK_ERR_SHAPE, "z-slabs need >= 2 planes each (mu halos are 2 deep)");
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
    const long long PL = nx * ny;
    // component stride: whole planes, rounded up to 64 doubles (512 B)
    e->slab.cstride = ((e->nzl + 2) * PL + 63) / 64 * 64;
    int rc = check_slab(&e->slab, vvl);
    if (rc) {
        delete e;
        return rc;
    }
    cudaGetDevice(&e->dev);
    const size_t dist_bytes = (size_t)e->slab.cstride * Q * sizeof(double);
    void *ptr = nullptr;
    for (int s = 0; s < 2; ++s)
        for (int d = 0; d < 2; ++d) {
            LTK_RC(engine_alloc(&ptr, dist_bytes, e));
            e->fg[s][d] = (double *)ptr;
        }
    LTK_RC(engine_alloc(&ptr, (size_t)(e->nzl + 2) * PL * sizeof(double), e));
    e->phi = (double *)ptr;
    // mu followed by the stress form's 4 aux arrays, one allocation
    e->mu_stride = ((e->nzl + 4) * PL + 63) / 64 * 64;
    LTK_RC(engine_alloc(&ptr, 5 * (size_t)e->mu_stride * sizeof(double), e));
    e->mu = (double *)ptr;
    LTK_RC(engine_alloc(&ptr, 2 * sizeof(long long), e));
    e->err = (long long *)ptr;
    LTK_RC(engine_alloc(&ptr, 2 * sizeof(unsigned long long), e));
    e->inbox = (unsigned long long *)ptr;
    // row-blocked f/g by default (measured faster, bitwise identical: DESIGN.md §4);
    // SoA for odd nx (16-byte rows) or LTK_LAYOUT=0
    e->lay = nx % 2 == 0 ? row_lay(&e->slab) : soa_lay(&e->slab);
    if (const char *v = getenv("LTK_LAYOUT"))
        if (atoi(v) == LTK_LAYOUT_SOA) e->lay = soa_lay(&e->slab);
    if (const char *v = getenv("LTK_PEER_OVERLAP")) e->peer_overlap = atoi(v) != 0;
    if (cudaStreamCreateWithFlags(&e->st, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&e->comm_st, cudaStreamNonBlocking) != cudaSuccess) {
        ltk_fluid_destroy(e);
        return fail(LTK_ERR_DEVICE, "stream creation failed");
    }
    for (int k = 0; k < 3; ++k) {
        cudaEventCreateWithFlags(&e->ev_fork[k], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&e->ev_join[k], cudaEventDisableTiming);
    }
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
    for (void *p : {(void *)e->inbox, (void *)e->err, (void *)e->phi, (void *)e->mu,
                    (void *)e->face})
        if (p) cudaFree(p);
    for (auto &s : e->fg)
        for (auto &p : s)
            if (p) cudaFree(p);
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
    if (phi) *phi = e->phi;  // phi / mu of the last step's input state
    if (mu) *mu = e->mu;
    return LTK_OK;
}

int ltk_fluid_stream(const ltk_fluid *e, void **stream) {
    *stream = e->st;
    return LTK_OK;
}

int ltk_fluid_set_params(ltk_fluid *e, const ltk_fluid_params *p) {
    LTK_RC(check_params(p));
    e->prm = *p;
    drop_graphs(e);
    return LTK_OK;
}

int ltk_fluid_load(ltk_fluid *e, const double *f_src, const double *g_src, int64_t padded,
                   int64_t nz_src, int64_t z_src0, void *stream) {
    if (e->failed) return fail(LTK_ERR_DEVICE, "engine failed (peer progress timeout)");
    cudaStream_t st = stream ? as_stream(stream) : e->st;
    if (e->transport == kPeer) LTK_RC(peer_before_load(e, st));
    e->cur = 0;
    LTK_RC(transpose(&e->slab, e->lay, e->fg[0][0], const_cast<double *>(f_src), padded, nz_src,
                     z_src0, Q, true, st));
    LTK_RC(transpose(&e->slab, e->lay, e->fg[0][1], const_cast<double *>(g_src), padded, nz_src,
                     z_src0, Q, true, st));
    if (e->transport == kLocal) LTK_RC(wrap_halos(&e->slab, e->lay, e->fg[0][0], e->fg[0][1],
                                                  nullptr, nullptr, 1, st));
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
    return LTK_OK;
}

int ltk_fluid_run(ltk_fluid *e, int64_t nsteps, void *stream) {
    if (e->failed) return fail(LTK_ERR_DEVICE, "engine failed (peer progress timeout)");
    cudaStream_t st = stream ? as_stream(stream) : e->st;
    for (int64_t k = 0; k < nsteps; ++k) {
        const int s = e->cur;
        if (e->prof) {
            for (int j = 0; j < 4; ++j) {
                cudaEvent_t ev;
                LTK_CUDA(cudaEventCreate(&ev));
                e->ppool.push_back(ev);
                e->pev[j] = ev;
            }
            LTK_RC(enqueue_step(e, s, st));
        } else if (e->use_graph && e->transport == kLocal) {
            if (!e->gexec[s]) {  // one graph per input state
                cudaGraph_t g;
                LTK_CUDA(cudaStreamBeginCapture(e->st, cudaStreamCaptureModeThreadLocal));
                int rc = enqueue_step(e, s, e->st);
                cudaError_t ce = cudaStreamEndCapture(e->st, &g);
                if (rc) return rc;
                if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture");
                ce = cudaGraphInstantiate(&e->gexec[s], g, 0);
                cudaGraphDestroy(g);
                if (ce != cudaSuccess) return cuda_fail(ce, "cudaGraphInstantiate");
            }
            LTK_CUDA(cudaGraphLaunch(e->gexec[s], st));
            count_launch(e->prm.physics >= 1 ? 3 : 2);
        } else {
            LTK_RC(enqueue_step(e, s, st));
        }
        e->cur = 1 - s;
        ++e->step;
    }
    return LTK_OK;
}

// Wait for the engine's streams, then read and clear its error words.
// LTK_ERR_SINGULAR (+ the lowest site in host order) when a kernel met
// rho <= 0; LTK_ERR_DEVICE when a peer progress wait timed out (the engine
// then refuses further steps: its halos may be stale).
int ltk_fluid_sync(ltk_fluid *e, int64_t *site) {
    *site = -1;
    LTK_CUDA(cudaStreamSynchronize(e->comm_st));
    LTK_CUDA(cudaStreamSynchronize(e->st));
    long long v[2] = {0, 0};
    LTK_CUDA(cudaMemcpyAsync(v, e->err, sizeof v, cudaMemcpyDeviceToHost, e->st));
    LTK_CUDA(cudaStreamSynchronize(e->st));
    if (v[1] != 0) {
        e->failed = true;
        return fail(LTK_ERR_DEVICE,
                    "peer progress wait timed out on rank %d: a neighbour slab stalled, "
                    "halos are stale", e->rank);
    }
    if (v[0] != 0) {
        LTK_CUDA(cudaMemsetAsync(e->err, 0, sizeof(long long), e->st));
        LTK_CUDA(cudaStreamSynchronize(e->st));
        *site = LLONG_MAX - v[0];
        return fail(LTK_ERR_SINGULAR, "rho <= 0 at lattice site %lld", (long long)*site);
    }
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
    long long SY, cstride, mu_stride;  // layout of the exporting slab
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
    b.cstride = e->slab.cstride;
    b.mu_stride = e->mu_stride;
    memset(blob, 0, LTK_IPC_BLOB_BYTES);
    memcpy(blob, &b, sizeof b);
    return LTK_OK;
}

static int open_peer(ltk_fluid *e, const char *blob, ltk_fluid::Peer &p) {
    IpcBlob b;
    memcpy(&b, blob, sizeof b);
    if (b.SY != e->lay.SY || b.cstride != e->slab.cstride || b.mu_stride != e->mu_stride)
        return fail(LTK_ERR_SHAPE, "peer slabs differ in layout");
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
    p.phi = (double *)ptrs[4];
    p.mu = (double *)ptrs[5];
    p.inbox = (unsigned long long *)ptrs[6];
    return LTK_OK;
}

static int attach_common(ltk_fluid *e) {
    if (e->nranks < 2) return fail(LTK_ERR_CONFIG, "a transport needs >= 2 slabs");
    if (e->transport != kLocal) return fail(LTK_ERR_CONFIG, "transport already attached");
    return preload_step_kernels();
}

static int attach_finish(ltk_fluid *e) {
    // complete before returning: the memsets must not land after a
    // neighbour's first progress signal (the caller barriers after attach)
    LTK_CUDA(cudaMemsetAsync(e->inbox, 0, 2 * sizeof(unsigned long long), e->st));
    LTK_CUDA(cudaMemsetAsync(e->err, 0, 2 * sizeof(long long), e->st));
    LTK_CUDA(cudaStreamSynchronize(e->st));
    e->transport = kPeer;
    drop_graphs(e);
    return LTK_OK;
}

int ltk_fluid_attach_peers(ltk_fluid *e, const char *up_blob, const char *dn_blob) {
    LTK_RC(attach_common(e));
    LTK_RC(open_peer(e, up_blob, e->up));
    if (memcmp(up_blob, dn_blob, sizeof(IpcBlob)) == 0)
        e->dn = e->up;  // two slabs: both neighbours are the same rank
    else
        LTK_RC(open_peer(e, dn_blob, e->dn));
    return attach_finish(e);
}

static void peer_from_engine(ltk_fluid::Peer &p, const ltk_fluid *o) {
    for (int st = 0; st < 2; ++st)
        for (int d = 0; d < 2; ++d) p.fg[st][d] = o->fg[st][d];
    p.phi = o->phi;
    p.mu = o->mu;
    p.inbox = o->inbox;
}

int ltk_fluid_attach_peer_engines(ltk_fluid *e, const ltk_fluid *up, const ltk_fluid *dn) {
    if (up->slab.cstride != e->slab.cstride || dn->slab.cstride != e->slab.cstride ||
        up->lay.SY != e->lay.SY || dn->lay.SY != e->lay.SY)
        return fail(LTK_ERR_SHAPE, "peer slabs differ in layout");
    LTK_RC(attach_common(e));
    peer_from_engine(e->up, up);
    peer_from_engine(e->dn, dn);
    return attach_finish(e);
}

int ltk_fluid_peer_timeout(ltk_fluid *e, int32_t *timed_out) {
    LTK_CUDA(cudaStreamSynchronize(e->st));
    LTK_CUDA(cudaStreamSynchronize(e->comm_st));
    long long v = 0;
    LTK_CUDA(cudaMemcpy(&v, e->err + 1, sizeof v, cudaMemcpyDeviceToHost));
    *timed_out = v != 0;
    return LTK_OK;
}

// Test hook: make this engine's next progress waits fail at once, as if a
// neighbour had stalled (the timeout path without an 8 s spin).
int ltk_fluid_inject_peer_timeout(ltk_fluid *e) {
    const long long one = 1;
    LTK_CUDA(cudaMemcpyAsync(e->err + 1, &one, sizeof one, cudaMemcpyHostToDevice, e->st));
    LTK_CUDA(cudaStreamSynchronize(e->st));
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
    if (e->transport != kLocal) return fail(LTK_ERR_CONFIG, "transport already attached");
    if (e->nzl < 2) return fail(LTK_ERR_SHAPE, "NCCL slabs need >= 2 planes (mu halos are 2 deep)");
    void *ptr = nullptr;
    LTK_RC(ltk_malloc(&ptr, 4 * 10 * (size_t)(e->nx * e->ny) * sizeof(double)));
    e->face = (double *)ptr;
    ncclUniqueId u;
    memcpy(u.internal, id, 128);
    LTK_NCCL(nccl().CommInitRank(&e->comm, e->nranks, u, e->rank));
    e->transport = kNccl;
    drop_graphs(e);
    return LTK_OK;
}

int ltk_fluid_set_layout(ltk_fluid *e, int32_t layout, int32_t *previous) {
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
    drop_graphs(e);
    return LTK_OK;
}

}  // extern "C"
