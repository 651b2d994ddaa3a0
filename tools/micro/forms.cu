// Issue cost of DFMA by operand form, mixed with K FFMA per DFMA (8 chains x 4 warps / scheduler).
// nvcc -O3 -arch=sm_100a forms.cu -o forms   (experiment, not part of the product)
#include <cstdio>
#include <cuda_runtime.h>

template <int FORM, int K>
__global__ void k(double* out, long long* cyc, int iters, double a, double b, float fa, const double* gp) {
    double d[8]; float f[8];
    double x = gp[threadIdx.x & 7], y = gp[8 + (threadIdx.x & 7)];  // register operands
#pragma unroll
    for (int i = 0; i < 8; ++i) { d[i] = a + threadIdx.x * 1e-3 + i; f[i] = (float)d[i]; }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (FORM == 0) d[i] = fma(d[i], x, y);        // 3 register pairs
            if (FORM == 1) d[i] = fma(d[i], a, y);        // reg, const, reg
            if (FORM == 2) d[i] = fma(d[i], x, b);        // reg, reg, const
            if (FORM == 3) d[i] = fma(d[i], d[i], b);     // same reg twice + const
            if (FORM == 4) d[i] = d[i] * a;               // DMUL reg, const
            if (FORM == 5) d[i] = d[i] + b;               // DADD reg, const
            if (FORM == 6) d[i] = fma(d[i], d[(i + 1) & 7], d[(i + 2) & 7]);  // 3 varying register pairs
            if (FORM == 7) d[i] = fma(d[i], 0.375, y);    // immediate
#pragma unroll
            for (int j = 0; j < K; ++j) f[i] = fmaf(f[i], fa, 1e-3f);
        }
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += d[i] + f[i];
    if (s == 123456.789) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int FORM, int K>
void run(const char* name, double* out, long long* cyc, double* gp) {
    const int iters = 2000, threads = 512;
    k<FORM, K><<<1, threads>>>(out, cyc, iters, 1.0000001, 1e-9, 1.0001f, gp);
    k<FORM, K><<<1, threads>>>(out, cyc, iters, 1.0000001, 1e-9, 1.0001f, gp);
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-22s K=%d: %.2f clk per {D-op + K FFMA} per scheduler\n", name, K, (double)h / (iters * 8.0) / 4);
}
#define ALLK(F, N) run<F, 0>(N, out, cyc, gp); run<F, 1>(N, out, cyc, gp); run<F, 2>(N, out, cyc, gp); run<F, 3>(N, out, cyc, gp);
int main() {
    double* out; long long* cyc; double* gp; cudaMalloc(&out, 64); cudaMalloc(&cyc, 8); cudaMalloc(&gp, 128);
    double h[16]; for (int i = 0; i < 16; ++i) h[i] = 1.0 + 1e-9 * i; cudaMemcpy(gp, h, 128, cudaMemcpyHostToDevice);
    ALLK(0, "DFMA r,r,r") ALLK(1, "DFMA r,c,r") ALLK(2, "DFMA r,r,c") ALLK(3, "DFMA r,r(same),c")
    ALLK(4, "DMUL r,c") ALLK(5, "DADD r,c") ALLK(6, "DFMA r,r',r'' varying") ALLK(7, "DFMA r,imm,r")
    return 0;
}
