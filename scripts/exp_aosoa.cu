// exp_aosoa.cu -- layout experiment for DESIGN.md §8 (not part of libltk.so).
//
// Question: k_collide_stream slows as a component plane grows past a 2 MB page
// (profiles/r01_plane_size_sweep.txt).  Hypothesis: with component-major SoA
// every SM touches ~79 component planes = ~79 pages at once.  Here the same
// pull + FAST forced collision runs over two layouts of random state:
//   SoA   : [comp][z][y][x]             (the engine's layout)
//   RowSoA: [z][y][comp][x]             (the 19 components of one x-row adjacent)
// at equal site counts and several plane sizes; mu is a plane-major array in both.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 exp_aosoa.cu -o exp_aosoa
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int Q = 19;
__constant__ int CX[Q] = {0, 1, -1, 0, 0, 0, 0, 1, 1, -1, -1, 1, 1, -1, -1, 0, 0, 0, 0};
__constant__ int CY[Q] = {0, 0, 0, 1, -1, 0, 0, 1, -1, 1, -1, 0, 0, 0, 0, 1, 1, -1, -1};
__constant__ int CZ[Q] = {0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1};
__constant__ double W[Q] = {1. / 3, 1. / 18, 1. / 18, 1. / 18, 1. / 18, 1. / 18, 1. / 18,
                            1. / 36, 1. / 36, 1. / 36, 1. / 36, 1. / 36, 1. / 36,
                            1. / 36, 1. / 36, 1. / 36, 1. / 36, 1. / 36, 1. / 36};

__device__ __forceinline__ int wrapi(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

// index of component i at (x, y, zs) (zs = storage plane incl. halos)
template <bool ROW>
__device__ __forceinline__ long long idx(int i, int x, int y, int zs, int nx, int ny, long long cstride) {
    if (ROW) return (((long long)zs * ny + y) * Q + i) * nx + x;
    return (long long)i * cstride + ((long long)zs * ny + y) * nx + x;
}

template <bool ROW>
__global__ void __launch_bounds__(128, 4) k_cs(const double *__restrict__ f, const double *__restrict__ g,
                                               const double *__restrict__ mu, double *fo, double *go, int nx,
                                               int ny, int nz, long long cstride) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)nx * ny * nz) return;
    const int x = (int)(t % nx), y = (int)((t / nx) % ny), z = (int)(t / ((long long)nx * ny));
    double F[Q], G[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        const long long s = idx<ROW>(i, wrapi(x - CX[i], nx), wrapi(y - CY[i], ny), z + 1 - CZ[i], nx, ny, cstride);
        F[i] = __ldg(f + s);
        G[i] = __ldg(g + s);
    }
    const long long PL = (long long)nx * ny, c = (long long)(z + 1) * PL + (long long)y * nx + x;
    const double m = __ldg(mu + c);
    const double gx = (__ldg(mu + c - x + wrapi(x + 1, nx)) - __ldg(mu + c - x + wrapi(x - 1, nx))) * 0.5;
    const double gy = (__ldg(mu + c + (long long)(wrapi(y + 1, ny) - y) * nx) -
                       __ldg(mu + c + (long long)(wrapi(y - 1, ny) - y) * nx)) * 0.5;
    const double gz = (__ldg(mu + c + PL) - __ldg(mu + c - PL)) * 0.5;
    double rho = 0, jx = 0, jy = 0, jz = 0, phi = 0;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        rho += F[i];
        jx += CX[i] * F[i];
        jy += CY[i] * F[i];
        jz += CZ[i] * F[i];
        phi += G[i];
    }
    const double Fx = -phi * gx, Fy = -phi * gy, Fz = -phi * gz, inv = 1.0 / rho;
    const double ux = fma(0.5, Fx, jx) * inv, uy = fma(0.5, Fy, jy) * inv, uz = fma(0.5, Fz, jz) * inv;
    const double usq = ux * ux + uy * uy + uz * uz, uF = ux * Fx + uy * Fy + uz * Fz;
    const double psi = m - phi / 3.0;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        const double ud = CX[i] * ux + CY[i] * uy + CZ[i] * uz, cF = CX[i] * Fx + CY[i] * Fy + CZ[i] * Fz;
        const double br = 1 + 3 * ud + 4.5 * ud * ud - 1.5 * usq;
        const double lam = i ? W[i] * 3.0 : -(1 - W[0]) * 3.0;
        const double fn = F[i] + (W[i] * rho * br - F[i]) + 0.5 * W[i] * (3 * (cF - uF) + 9 * ud * cF);
        const double gn = W[i] * phi * br + lam * psi;
        const long long o = idx<ROW>(i, x, y, z + 1, nx, ny, cstride);
        fo[o] = fn;
        go[o] = gn;
    }
}

template <bool ROW>
static float run(int nx, int ny, int nz, int iters) {
    const long long PL = (long long)nx * ny, planes = nz + 2;
    const long long cstride = (planes * PL + 63) / 64 * 64;
    const size_t dist = (size_t)Q * cstride * 8;
    double *f, *g, *fo, *go, *mu;
    cudaMalloc(&f, dist);
    cudaMalloc(&g, dist);
    cudaMalloc(&fo, dist);
    cudaMalloc(&go, dist);
    cudaMalloc(&mu, planes * PL * 8);
    std::vector<double> h(Q * cstride);
    for (size_t k = 0; k < h.size(); ++k) h[k] = (1.0 + 0.2 * ((k * 2654435761ull) % 1000) / 1000.0) / Q;
    cudaMemcpy(f, h.data(), dist, cudaMemcpyHostToDevice);
    cudaMemcpy(g, h.data(), dist, cudaMemcpyHostToDevice);
    cudaMemset(mu, 0, planes * PL * 8);
    const long long n = PL * nz;
    const unsigned grid = (unsigned)((n + 127) / 128);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int k = 0; k < 3; ++k) k_cs<ROW><<<grid, 128>>>(f, g, mu, fo, go, nx, ny, nz, cstride);
    cudaEventRecord(a);
    for (int k = 0; k < iters; ++k) {
        if (k & 1) k_cs<ROW><<<grid, 128>>>(fo, go, mu, f, g, nx, ny, nz, cstride);
        else k_cs<ROW><<<grid, 128>>>(f, g, mu, fo, go, nx, ny, nz, cstride);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaFree(f);
    cudaFree(g);
    cudaFree(fo);
    cudaFree(go);
    cudaFree(mu);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
    return ms / iters;
}

int main() {
    const int shapes[][3] = {{128, 128, 1024}, {256, 256, 256}, {512, 256, 128}, {512, 512, 64}, {1024, 256, 64}};
    printf("# same 16.8 M sites; ms per launch of the pull + FAST forced collision (616 B/site)\n");
    printf("# shape  plane_MB  SoA_ms  RowSoA_ms  SoA_TB/s  RowSoA_TB/s\n");
    for (auto &s : shapes) {
        const float a = run<false>(s[0], s[1], s[2], 20), b = run<true>(s[0], s[1], s[2], 20);
        const double bytes = 616.0 * s[0] * s[1] * s[2];
        printf("%dx%dx%d %.3f %.4f %.4f %.2f %.2f\n", s[0], s[1], s[2], s[0] * s[1] * 8.0 / (1 << 20), a, b,
               bytes / a / 1e9, bytes / b / 1e9);
    }
    return 0;
}
