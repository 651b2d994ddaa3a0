// Issue cost of {1 DFMA + A FFMA + B SHF (ALU) + C IMAD + D LDS} groups, 8 chains x 4 warps / scheduler.
// nvcc -O3 -arch=sm_100a forms2.cu -o forms2   (experiment, not part of the product)
#include <cstdio>
#include <cuda_runtime.h>

template <int ND, int A, int B, int C, int D>
__global__ void k(double* out, long long* cyc, int iters, double a, double b, float fa, unsigned ia) {
    __shared__ double sm[1024];
    double d[8]; float f[8]; unsigned n[8], m[8]; double l[8];
    sm[threadIdx.x] = threadIdx.x; sm[threadIdx.x + 512] = 1.0;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 8; ++i) { d[i] = a + threadIdx.x * 1e-3 + i; f[i] = (float)d[i]; n[i] = threadIdx.x * 7 + i; m[i] = n[i] * 3; l[i] = 0; }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
#pragma unroll
            for (int j = 0; j < ND; ++j) d[i] = fma(d[i], a, b);
#pragma unroll
            for (int j = 0; j < A; ++j) f[i] = fmaf(f[i], fa, 1e-3f);
#pragma unroll
            for (int j = 0; j < B; ++j) n[i] = __funnelshift_l(n[i], n[i], 3 + j);
#pragma unroll
            for (int j = 0; j < C; ++j) m[i] = m[i] * ia + (unsigned)it;
#pragma unroll
            for (int j = 0; j < D; ++j) l[i] += sm[(threadIdx.x + i * 32 + it) & 1023];
        }
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += d[i] + f[i] + n[i] + m[i] + l[i];
    if (s == 123456.789) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int ND, int A, int B, int C, int D>
void run(double* out, long long* cyc) {
    const int iters = 2000, threads = 512;
    k<ND, A, B, C, D><<<1, threads>>>(out, cyc, iters, 1.0000001, 1e-9, 1.0001f, 0x9e3779b1u);
    k<ND, A, B, C, D><<<1, threads>>>(out, cyc, iters, 1.0000001, 1e-9, 1.0001f, 0x9e3779b1u);
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%d DFMA + %d FFMA + %d SHF + %d IMAD + %d LDS(+DADD): %.2f clk per group per scheduler (%d instr)\n", ND, A, B, C, D,
           (double)h / (iters * 8.0) / 4, ND + A + B + C + 2 * D);
}
int main() {
    double* out; long long* cyc; cudaMalloc(&out, 64); cudaMalloc(&cyc, 8);
    run<1, 0, 0, 0, 0>(out, cyc);
    run<1, 1, 1, 0, 0>(out, cyc); run<1, 2, 1, 0, 0>(out, cyc); run<1, 3, 1, 0, 0>(out, cyc);
    run<1, 1, 0, 1, 0>(out, cyc); run<1, 0, 1, 1, 0>(out, cyc); run<1, 0, 0, 1, 0>(out, cyc); run<1, 0, 0, 2, 0>(out, cyc);
    run<2, 1, 1, 0, 0>(out, cyc); run<2, 2, 1, 0, 0>(out, cyc); run<2, 2, 2, 0, 0>(out, cyc); run<2, 1, 1, 1, 0>(out, cyc);
    run<2, 3, 1, 0, 0>(out, cyc); run<2, 2, 1, 1, 0>(out, cyc);
    run<0, 2, 0, 0, 0>(out, cyc); run<0, 2, 1, 0, 0>(out, cyc); run<0, 0, 0, 2, 0>(out, cyc); run<0, 1, 0, 1, 0>(out, cyc);
    run<2, 0, 0, 0, 1>(out, cyc); run<3, 1, 1, 0, 1>(out, cyc); run<0, 4, 0, 0, 0>(out, cyc);
    return 0;
}
