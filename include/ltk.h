/*
 * ltk.h -- C ABI of libltk.so, the B200 (sm_100a) implementation of the
 * targetDP lattice layer and the D3Q19 binary-fluid hot path.
 *
 * Plain C types only: device pointers are `double*` / `void*`, CUDA streams
 * and events are opaque `void*` (a cudaStream_t / cudaEvent_t; NULL = the
 * legacy default stream).  Every entry point returns an ltk_status; the
 * message of the last failure on the calling thread is ltk_last_error().
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference, the read-only upstream):
 *   memory    -> pkg/src/latkit/memory.py
 *   execution -> pkg/src/latkit/execution.py
 *   kernels   -> pkg/src/latkit/kernels.py
 * The full-timestep engine (ltk_fluid_*) has no reference counterpart: the
 * reference stops at the collision ("Collision only; no streaming step",
 * pkg/README.md:34-35); it implements the north-star extension of
 * SURVEY.md Appendix C, specified in DESIGN.md §2.
 */
#ifndef LTK_H
#define LTK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* libltk.so is built with -fvisibility=hidden; everything declared here is
 * the exported ABI. */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define LTK_ABI_VERSION 2
#define LTK_Q 19

typedef enum {
    LTK_OK = 0,
    LTK_ERR_CONFIG = 1,    /* -> ConfigError      (errors.py:12)  */
    LTK_ERR_BOUNDS = 2,    /* -> BoundsError      (errors.py:16)  */
    LTK_ERR_SHAPE = 3,     /* -> ShapeError       (errors.py:20)  */
    LTK_ERR_ALLOC = 4,     /* -> AllocationError  (errors.py:24)  */
    LTK_ERR_LIFECYCLE = 5, /* -> LifecycleError   (errors.py:28)  */
    LTK_ERR_PLAN = 6,      /* -> PlanError        (errors.py:32)  */
    LTK_ERR_DEVICE = 7,    /* -> DeviceError      (errors.py:36)  */
    LTK_ERR_SINGULAR = 11  /* -> SingularStateError (errors.py:52) */
} ltk_status;

/* Arithmetic mode of the collision.
 * EXACT: the reference op order, true IEEE divisions, no FMA contraction ->
 *        bitwise equal to reference kernels.py:89-125 (numba emits no FMA).
 * FAST:  hoisted reciprocals and FMA -> within 1e-12 relative of EXACT. */
typedef enum { LTK_MODE_EXACT = 0, LTK_MODE_FAST = 1 } ltk_mode;

/* ------------------------------------------------------------ runtime */

int ltk_abi_version(void);
const char *ltk_last_error(void);
int ltk_device_count(int *count);
int ltk_set_device(int device);
int ltk_get_device(int *device);
/* name: >= 256 bytes */
int ltk_device_info(int device, char *name, int *sm_count, int64_t *total_mem,
                    int *cc_major, int *cc_minor);

/* targetMalloc / targetFree (memory.py:231-253): zero-initialised device
 * allocation of `bytes`, 256-byte aligned. */
int ltk_malloc(void **ptr, size_t bytes);
int ltk_free(void *ptr);
int ltk_mem_info(size_t *free_bytes, size_t *total_bytes);
int ltk_memset0(void *ptr, size_t bytes, void *stream);

/* copyToTarget / copyFromTarget (memory.py:261-274), asynchronous on
 * `stream`; host memory should be pinned (ltk_host_register) for overlap. */
int ltk_h2d(void *dst, const void *src, size_t bytes, void *stream);
int ltk_d2h(void *dst, const void *src, size_t bytes, void *stream);
int ltk_d2d(void *dst, const void *src, size_t bytes, void *stream);
int ltk_host_register(void *ptr, size_t bytes);
int ltk_host_unregister(void *ptr);
int ltk_host_alloc(void **ptr, size_t bytes);
int ltk_host_free(void *ptr);

int ltk_stream_create(void **stream);
int ltk_stream_destroy(void *stream);
int ltk_stream_sync(void *stream);
int ltk_event_create(void **event, int timing);
int ltk_event_destroy(void *event);
int ltk_event_record(void *event, void *stream);
/* *done = 1 when the event has completed */
int ltk_event_query(void *event, int *done);
int ltk_event_sync(void *event);
int ltk_event_elapsed(void *start, void *stop, float *ms);
int ltk_stream_wait_event(void *stream, void *event);

/* syncTarget (execution.py:271-281): synchronise `stream`, then read and
 * clear the stream's error word (every stream has its own, so kernels of one
 * TargetDevice never report to another sharing the GPU).  Returns
 * LTK_ERR_SINGULAR (and the lowest offending real site in *site) when a
 * kernel launched on `stream` met rho <= 0 at a real lattice site
 * (kernels.py:106-108), else LTK_OK with *site = -1. */
int ltk_sync(void *stream, int64_t *site);

/* Kernels launched by this library since load (for the bench's
 * gpu_launches claim). */
int64_t ltk_launch_count(void);

/* ------------------------------------------------------------ kernels */

/* Replaces the range runner of scale_kernel, kernels.py:79-86:
 * field[c*padded + s] *= a for c < 3 and s in [chunk_lo*vvl, chunk_hi*vvl).
 * vvl in {1,2,4,8,16}; tpb = threads per block (LaunchPlan.tpb). */
int ltk_scale(int64_t chunk_lo, int64_t chunk_hi, int32_t vvl, int32_t tpb,
              double *field, int64_t padded, double a, void *stream);

/* Constants of the collision: the constant-store keys of
 * set_model_constants (kernels.py:194-200).  cv is not passed: the kernels
 * hard-code the canonical D3Q19 ordering (model.py:21-34) and the Python
 * prepare() rejects any other cv with ConfigError. */
typedef struct {
    double wv[LTK_Q];
    double cs2;
    double tau_f;
    double tau_g;
    int32_t mode; /* ltk_mode */
    int32_t reserved;
} ltk_collision_params;

/* Replaces _collision_range(chunk_lo, chunk_hi, vvl, f, g, padded, nsites,
 * wv, cvx, cvy, cvz, cs2, tau_f, tau_g), kernels.py:89-125: in-place binary
 * BGK collision of the SoA fields f, g ([19][padded] doubles, device) over
 * sites [chunk_lo*vvl, chunk_hi*vvl).  One CUDA thread per VVL-site chunk
 * (TLP), VVL consecutive sites per thread with vector loads (ILP).  Zero-
 * density padding sites are left untouched; rho <= 0 at a real site sets the
 * device error word reported by ltk_sync. */
int ltk_collide(int64_t chunk_lo, int64_t chunk_hi, int32_t vvl, int32_t tpb, double *f,
                double *g, int64_t padded, int64_t nsites, const ltk_collision_params *p,
                void *stream);

/* Masked transfers (memory.py:277-315): component-major pack of the k sites
 * listed in idx (device int64[k]) into packed[ncomp*k], and the inverse. */
/* Diagnostics: the EXACT-mode division (x * RN(1/d) with one FMA residual
 * correction, Markstein) next to the hardware IEEE division, element-wise
 * over device arrays x[n], d[n] (d > 0).  Test infrastructure for the claim
 * that EXACT mode stays bitwise equal to the reference's true divisions. */
int ltk_div_selftest(const double *x, const double *d, int64_t n, double *out_rcp,
                     double *out_div, void *stream);
int ltk_pack_sites(const double *src, double *packed, const int64_t *idx, int64_t k,
                   int32_t ncomp, int64_t padded, void *stream);
int ltk_unpack_sites(double *dst, const double *packed, const int64_t *idx, int64_t k,
                     int32_t ncomp, int64_t padded, void *stream);

/* ------------------------------------------------------------ full timestep
 * Builder-defined extension.
 *
 * Device layout of a slab: SoA, component stride `cstride`
 * doubles; inside a component, storage plane zs = z + 1 (z = 0..nzl-1 owned,
 * zs = 0 and zs = nzl+1 are halo planes), site (x, y) at zs*nx*ny + y*nx + x
 * (x fastest).  Periodic in x and y; z neighbours come from the halo planes.
 * phi arrays: (nzl+2)*nx*ny doubles, plane zs = z + 1 (one halo per face).
 * mu arrays: (nzl+4)*nx*ny doubles, plane zs = z + 2 (two halos per face:
 * the filtered potential force reads mu at z +- 2).
 */
typedef struct {
    double wv[LTK_Q];
    double lam[LTK_Q];  /* g_eq chemical-potential weights */
    double cs2, tau_f, tau_g;
    double A, B, kappa, gamma; /* mu = A phi + B phi^3 - kappa lap(phi); mobility gamma */
    int32_t physics;    /* 0 = passive (reference collision), 1 = free-energy binary fluid
                         * with the potential force -phi grad(mu), each component
                         * filtered [1/4 1/2 1/4] along its own axis,
                         * 2 = same with the momentum-conserving F = -div P
                         * (chemical pressure tensor; engine only) */
    int32_t mode;       /* ltk_mode */
} ltk_fluid_params;

typedef struct {
    int64_t nx, ny, nzl;  /* owned extent of this slab */
    int64_t cstride;      /* doubles between components (>= (nzl+2)*nx*ny) */
} ltk_slab;

/* phi(x) = sum_i g_i(x - c_i) on owned planes [z_lo, z_hi) (pull). */
int ltk_fluid_phi(const ltk_slab *s, const double *g, double *phi, int64_t z_lo,
                  int64_t z_hi, void *stream);
/* mu = A phi + B phi^3 - kappa lap7(phi) on owned planes [z_lo, z_hi);
 * phi needs its halo planes, mu is written in the two-halo mu layout. */
int ltk_fluid_mu(const ltk_slab *s, const double *phi, double *mu,
                 const ltk_fluid_params *p, int64_t z_lo, int64_t z_hi, void *stream);
/* Pull-stream + collide owned planes [z_lo, z_hi): f_out(x) = C(f_in(x-c_i), ...).
 * physics 1 reads phi (x, x+-1 per axis) and mu (x, x+-1, x+-2 per axis);
 * physics 0 ignores phi/mu; physics 2 runs in the engine only.  rho <= 0
 * sets the error word of `stream` (ltk_sync). */
int ltk_fluid_collide_stream(const ltk_slab *s, const double *f_in, const double *g_in,
                             const double *phi, const double *mu, double *f_out,
                             double *g_out, const ltk_fluid_params *p, int64_t z_lo,
                             int64_t z_hi, int32_t vvl, void *stream);
/* Periodic z wrap on one device: copy owned boundary planes into the halo
 * planes.  which: bit0 = f/g crossing components, bit1 = phi (1 plane per
 * face), bit2 = mu (2 planes per face). */
int ltk_fluid_wrap_halos(const ltk_slab *s, double *f, double *g, double *phi, double *mu,
                         int32_t which, void *stream);
/* Halo faces of the distributions: pack the 5 f + 5 g components that cross
 * the top (dir=+1: cz=+1 set, owned plane nzl-1) or bottom (dir=-1: cz=-1
 * set, owned plane 0) face into buf[10*nx*ny]; unpack writes such a buffer
 * into the opposite halo plane (dir=+1 -> halo zs=0, dir=-1 -> zs=nzl+1). */
int ltk_fluid_pack_face(const ltk_slab *s, const double *f, const double *g, double *buf,
                        int32_t dir, void *stream);
int ltk_fluid_unpack_face(const ltk_slab *s, double *f, double *g, const double *buf,
                          int32_t dir, void *stream);

/* Host-order <-> slab conversion: `host` is a device copy of
 * a reference-ordered SoA field ([ncomp][padded], site (x*ny+y)*nz+z over
 * the global lattice nx*ny*nz_global); the slab holds global planes
 * [z0, z0+nzl). */
int ltk_fluid_scatter(const ltk_slab *s, const double *host, int64_t padded,
                      int64_t nz_global, int64_t z0, int32_t ncomp, double *slab,
                      void *stream);
int ltk_fluid_gather(const ltk_slab *s, const double *slab, int64_t padded,
                     int64_t nz_global, int64_t z0, int32_t ncomp, double *host,
                     void *stream);

/* ---- engine: owns the slab buffers and runs whole timesteps in C++ ---- */
typedef struct ltk_fluid ltk_fluid;

/* Create a slab engine on the current device.  nranks == 1 -> periodic wrap
 * on one device; nranks > 1 -> halo exchange with ranks (rank+-1) mod
 * nranks, by peer stores from the kernels (ltk_fluid_attach_peers) or by
 * NCCL (ltk_fluid_attach_nccl).  vvl: sites per thread of the fused
 * collide-stream kernel. */
int ltk_fluid_create(int64_t nx, int64_t ny, int64_t nz_global, int32_t rank,
                     int32_t nranks, const ltk_fluid_params *p, int32_t vvl,
                     ltk_fluid **out);
int ltk_fluid_destroy(ltk_fluid *e);
int ltk_fluid_slab(const ltk_fluid *e, ltk_slab *s, int64_t *z0);
/* Device pointers of the current state (post-collision f, g) and of phi/mu.
 * f/g are in the engine's layout (ltk_fluid_set_layout: row-blocked by
 * default for even nx, not the ltk_slab SoA layout); ltk_fluid_store gives
 * them in host order.  phi/mu are plane-major (zs*nx*ny + y*nx + x). */
int ltk_fluid_buffers(const ltk_fluid *e, double **f, double **g, double **phi, double **mu);
int ltk_fluid_set_params(ltk_fluid *e, const ltk_fluid_params *p);
/* The engine's CUDA stream (all engine work is ordered on it). */
int ltk_fluid_stream(const ltk_fluid *e, void **stream);
/* Load/store the slab from/to a reference-ordered state that sits on the
 * device: src/dst are [19][padded] arrays over an nx*ny*nz_src lattice
 * (site (x*ny+y)*nz_src + z); this slab's plane 0 is plane z_src0 there.
 * Pass nz_src = nz_global, z_src0 = slab z0 for a full-lattice array, or
 * nz_src = nzl, z_src0 = 0 for an array holding only this slab. */
int ltk_fluid_load(ltk_fluid *e, const double *f_src, const double *g_src, int64_t padded,
                   int64_t nz_src, int64_t z_src0, void *stream);
int ltk_fluid_store(ltk_fluid *e, double *f_dst, double *g_dst, int64_t padded,
                    int64_t nz_src, int64_t z_src0, void *stream);
/* Diagnostics of the current state over this slab's owned sites:
 * out5 = {sum rho, sum j_x, sum j_y, sum j_z, sum phi} (synchronous;
 * deterministic block-tree order; sum over slabs for the whole lattice). */
int ltk_fluid_totals(ltk_fluid *e, double *out5);
/* Run n full timesteps on the engine stream (or `stream` if not NULL).
 * Asynchronous; errors surface at ltk_fluid_sync. */
int ltk_fluid_run(ltk_fluid *e, int64_t nsteps, void *stream);
/* syncTarget for an engine: wait for its streams, then read and clear its
 * own error words.  LTK_ERR_SINGULAR (+ lowest site in host order) when a
 * kernel met rho <= 0; LTK_ERR_DEVICE when a peer progress wait timed out
 * (a neighbour stalled: halos are stale, and the engine refuses further
 * loads and steps). */
int ltk_fluid_sync(ltk_fluid *e, int64_t *site);
/* Capture one step pair (A->B, B->A) into CUDA graphs used by ltk_fluid_run. */
int ltk_fluid_use_graph(ltk_fluid *e, int32_t enable);
/* Chemical-potential stencil kernel, process-wide.  LTK_MU_AUTO: the
 * shared-memory tile kernel k_mu_tile where it applies (nx % 32 == 0,
 * ny % 8 == 0), else k_mu; LTK_MU_PLAIN forces k_mu.  Bitwise identical.
 * variant < 0 only queries; *previous (if not NULL) gets the old value. */
#define LTK_MU_AUTO 0
#define LTK_MU_PLAIN 1
int ltk_fluid_mu_variant(int32_t variant, int32_t *previous);

/* f/g storage layout of an engine.  LTK_LAYOUT_SOA: component-major
 * planes, element (i, zs, y, x) at i*cstride + zs*nx*ny + y*nx + x -- the
 * ltk_slab layout every slab-level entry point above takes.  LTK_LAYOUT_ROW:
 * row-blocked, element at zs*ny*19*nx + (y*19 + i)*nx + x (the 19 components
 * of one x-row adjacent; even nx; the default of new engines with even nx,
 * measured ~1.5% faster on the full step).  Results are bitwise identical; only the
 * engine's own buffers change (ltk_fluid_buffers' f/g pointers then hold
 * that layout).  Set before ltk_fluid_load and before attaching a transport
 * (the state is undefined after a change); every transport works with
 * either layout (NCCL faces are packed); peer slabs must agree.  The
 * environment variable LTK_LAYOUT=0 makes SoA the default of new engines.  layout < 0 only queries (*previous).  Not in the reference: a
 * B200 layout choice. */
#define LTK_LAYOUT_SOA 0
#define LTK_LAYOUT_ROW 1
int ltk_fluid_set_layout(ltk_fluid *e, int32_t layout, int32_t *previous);
/* Last step's per-kernel device times in ms (phi, mu, collide_stream, halo). */
int ltk_fluid_profile(ltk_fluid *e, int32_t enable, float *ms4);

/* Peer transport (one node, NVLink/NVSwitch): every slab exports its buffers
 * with CUDA IPC (ltk_fluid_ipc_blob), the caller exchanges the blobs
 * (torch.distributed) and attaches the slabs above and below.  The boundary
 * planes' kernels then store their halo images directly into the neighbours'
 * buffers (peer stores over NVLink) and progress counters pushed into the
 * neighbours' inboxes order the phases -- the halo exchange is fused into the
 * producing kernels.  Call before ltk_fluid_load. */
#define LTK_IPC_BLOB_BYTES 1024
int ltk_fluid_ipc_blob(ltk_fluid *e, char *blob);
int ltk_fluid_attach_peers(ltk_fluid *e, const char *up_blob, const char *dn_blob);
/* Same transport between engines of one process (one thread driving several
 * GPUs, or several slabs on one GPU): peers given directly. */
int ltk_fluid_attach_peer_engines(ltk_fluid *e, const ltk_fluid *up, const ltk_fluid *dn);
/* 1 if a peer progress wait ever exceeded its budget (~8 s; never expected). */
int ltk_fluid_peer_timeout(ltk_fluid *e, int32_t *timed_out);
/* Test hook: the engine's next progress waits fail at once, as if a
 * neighbour had stalled. */
int ltk_fluid_inject_peer_timeout(ltk_fluid *e);

/* NCCL (dlopen'ed libnccl.so.2): the 128-byte unique id of rank 0 is
 * broadcast by the caller (torch.distributed) before attach. */
int ltk_nccl_available(void);
int ltk_nccl_unique_id(char id[128]);
int ltk_fluid_attach_nccl(ltk_fluid *e, const char id[128]);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* LTK_H */
