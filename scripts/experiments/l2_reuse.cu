// l2_reuse.cu -- how far back can a streaming kernel re-read what it wrote
// and still hit L2 on B200?  Models the g' re-read of the phi pass
// (DESIGN.md §4.3): chunk k of a stream reads 2 x C bytes (f, g of a plane),
// writes 2 x C bytes (f', g') and re-reads the g' chunk written `lag` chunks
// earlier (C bytes).  One kernel launch per chunk, in stream order.  Reported:
// ms per chunk; the re-read costs nothing extra when it hits L2.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_reuse l2_reuse.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void k_chunk(const double2 *__restrict__ fin, const double2 *__restrict__ gin,
                        double2 *__restrict__ fout, double2 *__restrict__ gout,
                        const double2 *__restrict__ gre, double2 *__restrict__ sink, long long n,
                        int reread) {
    double2 acc = make_double2(0.0, 0.0);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double2 a = fin[i], b = gin[i];
        fout[i] = make_double2(a.x * 1.000001, a.y);
        gout[i] = make_double2(b.x * 0.999999, b.y);
        if (reread) {
            double2 c = __ldcg(gre + i);
            acc.x += c.x;
            acc.y += c.y;
        }
    }
    if (acc.x == 12345.678) sink[0] = acc;  // keep the loads
}

int main(int argc, char **argv) {
    const double chunk_mb = argc > 1 ? atof(argv[1]) : 10.0;  // one g' plane at 256^2 ~ 10 MB
    const int nchunks = 256;
    const long long n = (long long)(chunk_mb * 1e6 / 16);     // double2 per chunk
    const size_t cb = n * sizeof(double2);
    double2 *fin, *gin, *fout, *gout, *sink;
    cudaMalloc(&fin, cb * nchunks);
    cudaMalloc(&gin, cb * nchunks);
    cudaMalloc(&fout, cb * nchunks);
    cudaMalloc(&gout, cb * nchunks);
    cudaMalloc(&sink, 64);
    cudaMemset(fin, 0, cb * nchunks);
    cudaMemset(gin, 0, cb * nchunks);
    cudaMemset(fout, 0, cb * nchunks);
    cudaMemset(gout, 0, cb * nchunks);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int lags[] = {-1, 1, 2, 3, 4, 6, 8, 12, 16, 24};
    printf("# chunk %.1f MB: per chunk read 2C + write 2C (+ re-read C of chunk k-lag)\n", chunk_mb);
    for (int li = 0; li < (int)(sizeof lags / sizeof lags[0]); ++li) {
        const int lag = lags[li];
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            for (int k = 0; k < nchunks; ++k) {
                const int kr = lag > 0 ? (k >= lag ? k - lag : k + nchunks - lag) : 0;
                k_chunk<<<nsm * 8, 256>>>(fin + k * n, gin + k * n, fout + k * n, gout + k * n,
                                          gout + (long long)kr * n, sink, n, lag > 0);
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep == 1) {
                const double base = 4.0 * cb;
                const double tot = base + (lag > 0 ? cb : 0);
                printf("lag %3d (reuse distance %6.0f MB): %.4f ms/chunk, %.0f GB/s counting the "
                       "re-read, %.0f GB/s without it\n",
                       lag, lag > 0 ? lag * 5.0 * chunk_mb : 0.0, ms / nchunks,
                       tot * nchunks / (ms * 1e-3) / 1e9, base * nchunks / (ms * 1e-3) / 1e9);
            }
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
