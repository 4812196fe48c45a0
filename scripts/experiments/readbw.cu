// Pure HBM read bandwidth (16-byte loads, 4 in flight per thread, grid of
// 148 x k blocks): the ceiling for read-dominated kernels such as k_phi.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const double2 *__restrict__ p, long long n2, double *out) {
    double acc = 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n2; i += 4 * stride) {
        double2 a = __ldg(p + i), b = __ldg(p + i + stride), c = __ldg(p + i + 2 * stride),
                d = __ldg(p + i + 3 * stride);
        acc += a.x + a.y + b.x + b.y + c.x + c.y + d.x + d.y;
    }
    for (; i < n2; i += stride) acc += __ldg(p + i).x;
    if (acc == 123.456) out[0] = acc;
}
int main() {
    const long long n = 19LL * 256 * 256 * 256, n2 = n / 2;
    double *p, *o;
    cudaMalloc(&p, n * 8);
    cudaMalloc(&o, 8);
    cudaMemset(p, 0, n * 8);
    cudaEvent_t s, e;
    cudaEventCreate(&s);
    cudaEventCreate(&e);
    for (int k : {4, 8, 16, 32}) {
        float best = 1e9;
        for (int r = 0; r < 8; ++r) {
            cudaEventRecord(s);
            rd<<<148 * k, 256>>>((const double2 *)p, n2, o);
            cudaEventRecord(e);
            cudaEventSynchronize(e);
            float ms;
            cudaEventElapsedTime(&ms, s, e);
            if (ms < best) best = ms;
        }
        printf("blocks/SM %2d: read %.0f GB/s\n", k, n * 8 / best / 1e6);
    }
    return 0;
}
