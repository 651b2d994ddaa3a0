// Dependent-issue latency of the instructions on the cost kernel's critical chains, and FP64
// pipe utilisation versus (warps per scheduler) x (independent chains per warp).
// nvcc -O3 -arch=sm_100a lat.cu -o lat   (not part of the product)
#include <cstdio>
#include <cuda_runtime.h>

template <int CH, int OP>
__global__ void k(double* out, long long* cyc, int iters, double a, double b) {
    double d[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) d[i] = a + threadIdx.x * 1e-3 + i;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int i = 0; i < CH; ++i) {
                if (OP == 0) d[i] = fma(d[i], a, b);
                if (OP == 1) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d[i])); d[i] = y; }
                if (OP == 2) { float f = __double2float_rn(d[i]); d[i] = __hiloint2double(__float_as_int(f), 0); }
                if (OP == 3) { d[i] = d[i] > b ? a : d[i]; }
            }
        }
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += d[i];
    if (s == 123456.789) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int CH, int OP>
void run(const char* name, int threads, double* out, long long* cyc) {
    const int iters = 2000;
    k<CH, OP><<<1, threads>>>(out, cyc, iters, 1.0000001, 1e-9);
    k<CH, OP><<<1, threads>>>(out, cyc, iters, 1.0000001, 1e-9);
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double per = (double)h / (iters * 8.0);
    printf("%-10s warps/SMSP %d chains %d: %.2f cycles per round of %d (%.2f cyc/instr/SMSP-warp; pipe busy %.0f%% if 2 cyc/instr)\n", name,
           threads / 128 ? threads / 128 : 1, CH, per, CH, per / CH, OP == 0 ? 100.0 * (threads >= 128 ? threads / 128 : 1) * CH * 2.0 / per : 0.0);
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 64); cudaMalloc(&cyc, 8);
    for (int threads : {32, 128, 256, 512, 768}) {
        run<1, 0>("DFMA", threads, out, cyc); run<2, 0>("DFMA", threads, out, cyc); run<4, 0>("DFMA", threads, out, cyc);
        run<8, 0>("DFMA", threads, out, cyc);
    }
    run<1, 1>("RSQ64H", 32, out, cyc); run<4, 1>("RSQ64H", 32, out, cyc);
    run<1, 2>("D2F", 32, out, cyc); run<4, 2>("D2F", 32, out, cyc);
    run<1, 3>("DSETP+SEL", 32, out, cyc);
    return 0;
}
