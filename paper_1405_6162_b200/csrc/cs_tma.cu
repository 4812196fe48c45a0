// cs_tma.cu -- launchers of k_cs_tma (cs_tma.cuh): the tile geometry per
// lattice width and the template instances.
#include <cstdlib>

#include "cs_tma.cuh"

namespace ltk {

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

template <int MODE, int PHYS, int T1, int TX, bool FULL, int STAGES, int NCW, int NPW>
static int launch_cfg(const FluidArgs &a, cudaStream_t st) {
    using Gm = TmaGeom<TX, FULL>;
    constexpr size_t smem = STAGES * Gm::stage_bytes;
    static_assert(smem <= 227 * 1024, "stage ring exceeds shared memory");
    auto kern = k_cs_tma<MODE, PHYS, T1, TX, FULL, STAGES, NCW, NPW>;
    static bool attr = false;
    if (!attr) {
        LTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    const long long ntiles = a.nthreads / TX;
    const unsigned grid = (unsigned)std::min<long long>(ntiles, num_sms());
    kern<<<grid, 32 * ((NPW > 0 ? NPW : 1) + NCW), smem, st>>>(a);
    LTK_CHECK_LAUNCH("k_cs_tma");
    return LTK_OK;
}

// Loader (env LTK_TMA_LOADER): 0 = TMA bulk row copies (default), 1 = LDGSTS.
// Measured at 256^3 FAST: 1.755 ms (TMA) / 2.21 ms (LDGSTS) per launch vs
// 1.555 ms for k_collide_stream (profiles/r01_cs_tma.md).
static int loader() {
    static const int v = getenv("LTK_TMA_LOADER") ? atoi(getenv("LTK_TMA_LOADER")) : 0;
    return v;
}

template <int MODE, int PHYS, int T1, int TX, bool FULL, int STAGES>
static int launch_ld(const FluidArgs &a, cudaStream_t st) {
    if (loader() == 0) return launch_cfg<MODE, PHYS, T1, TX, FULL, STAGES, 11, 0>(a, st);
    return launch_cfg<MODE, PHYS, T1, TX, FULL, STAGES, 11, 4>(a, st);
}

template <int MODE, int PHYS, int T1>
static int launch_t(const FluidArgs &a, cudaStream_t st) {
    if (a.nx == 128) return launch_ld<MODE, PHYS, T1, 128, true, 4>(a, st);
    if (a.nx == 256) return launch_ld<MODE, PHYS, T1, 256, true, 2>(a, st);
    if (a.nx % 256 == 0) return launch_ld<MODE, PHYS, T1, 256, false, 2>(a, st);
    return launch_ld<MODE, PHYS, T1, 128, false, 4>(a, st);
}

// Module preload for the peer transport (see fluid.cu preload_step_kernels):
// every instance launch_t can pick for this lattice width.
template <int MODE, int PHYS, int T1, int TX, bool FULL, int STAGES>
static void preload_ld() {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_cs_tma<MODE, PHYS, T1, TX, FULL, STAGES, 11, 0>);
    cudaFuncGetAttributes(&fa, k_cs_tma<MODE, PHYS, T1, TX, FULL, STAGES, 11, 4>);
}

template <int MODE, int PHYS, int T1>
static void preload_t(int nx) {
    if (nx == 128) preload_ld<MODE, PHYS, T1, 128, true, 4>();
    else if (nx == 256) preload_ld<MODE, PHYS, T1, 256, true, 2>();
    else if (nx % 256 == 0) preload_ld<MODE, PHYS, T1, 256, false, 2>();
    else if (nx % 128 == 0) preload_ld<MODE, PHYS, T1, 128, false, 4>();
}

void preload_cs_tma(int nx) {
    preload_t<LTK_MODE_FAST, 0, 0>(nx);
    preload_t<LTK_MODE_FAST, 1, 0>(nx);
    preload_t<LTK_MODE_EXACT, 0, 0>(nx);
    preload_t<LTK_MODE_EXACT, 0, 1>(nx);
    preload_t<LTK_MODE_EXACT, 0, 2>(nx);
    preload_t<LTK_MODE_EXACT, 0, 3>(nx);
    preload_t<LTK_MODE_EXACT, 1, 0>(nx);
    preload_t<LTK_MODE_EXACT, 1, 1>(nx);
    preload_t<LTK_MODE_EXACT, 1, 2>(nx);
    preload_t<LTK_MODE_EXACT, 1, 3>(nx);
}

bool cs_tma_ok(const FluidArgs &a, int vvl) {
    return vvl == 1 && a.nx % 128 == 0 && a.nthreads > 0 && a.SI == a.cstride;  // SoA only
}

int launch_cs_tma(const FluidArgs &a, int mode, int phys, cudaStream_t st) {
    const int t1 = (a.tau_f == 1.0 ? 1 : 0) | (a.tau_g == 1.0 ? 2 : 0);
    if (mode == LTK_MODE_FAST) {
        return phys == 1 ? launch_t<LTK_MODE_FAST, 1, 0>(a, st) : launch_t<LTK_MODE_FAST, 0, 0>(a, st);
    }
    if (phys == 1) {
        switch (t1) {
            case 0: return launch_t<LTK_MODE_EXACT, 1, 0>(a, st);
            case 1: return launch_t<LTK_MODE_EXACT, 1, 1>(a, st);
            case 2: return launch_t<LTK_MODE_EXACT, 1, 2>(a, st);
            default: return launch_t<LTK_MODE_EXACT, 1, 3>(a, st);
        }
    }
    switch (t1) {
        case 0: return launch_t<LTK_MODE_EXACT, 0, 0>(a, st);
        case 1: return launch_t<LTK_MODE_EXACT, 0, 1>(a, st);
        case 2: return launch_t<LTK_MODE_EXACT, 0, 2>(a, st);
        default: return launch_t<LTK_MODE_EXACT, 0, 3>(a, st);
    }
}

}  // namespace ltk
