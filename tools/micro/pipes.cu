// Pipe-throughput and seed-precision microbenchmarks that inform the cost kernel's
// instruction selection (not part of the product).  nvcc -O3 -arch=sm_100a pipes.cu -o pipes
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

#define CHAINS 8
enum { DFMA, DADD, DMUL, D2F, F2D, RCP64, RSQ64, F2I, FFMA, DFMA_FFMA, DFMA_IADD, DSETSEL, DFMA_LDS, FFMA_IADD,
       DFMA_D2F, DFMA_MUFU, I2D, D2I, DMNMX, NOPS };
const char* NAMES[] = {"DFMA", "DADD", "DMUL", "F2F.F32.F64", "F2F.F64.F32", "MUFU.RCP64H", "MUFU.RSQ64H", "F2I.F32",
                       "FFMA", "DFMA+FFMA 1:1", "DFMA+IADD 1:1", "DSETP+SEL", "DFMA+LDS64 1:1", "FFMA+IADD 1:1",
                       "DFMA+D2F 4:1", "DFMA+MUFU64 4:1", "I2F.F64.S32", "F2I.S32.F64", "DMNMX(fmax)"};

template <int OP>
__global__ void k(double* out, int iters, double a, double b) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = a + i * 1e-9;
    __syncthreads();
    double d[CHAINS];
    float f[CHAINS];
    int n[CHAINS];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) { d[i] = a + threadIdx.x * 1e-3 + i; f[i] = (float)d[i]; n[i] = threadIdx.x + i; }
    const float fa = (float)a, fb = (float)b;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) {
            if (OP == DFMA) d[i] = fma(d[i], a, b);
            if (OP == DADD) d[i] = d[i] + b;
            if (OP == DMUL) d[i] = d[i] * a;
            if (OP == D2F) { f[i] = __double2float_rn(d[i]); d[i] = __hiloint2double(__float_as_int(f[i]) + 0x3ff00000, n[i]); }
            if (OP == F2D) { d[i] = (double)f[i]; f[i] = __int_as_float(__double2hiint(d[i]) ^ __double2loint(d[i])); }
            if (OP == RCP64) { double y; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d[i])); d[i] = y; }
            if (OP == RSQ64) { double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d[i])); d[i] = y; }
            if (OP == F2I) { n[i] = __float2int_rz(f[i]); f[i] = __int_as_float(n[i] | 0x3f800000); }
            if (OP == FFMA) f[i] = fmaf(f[i], fa, fb);
            if (OP == DFMA_FFMA) { d[i] = fma(d[i], a, b); f[i] = fmaf(f[i], fa, fb); }
            if (OP == DFMA_IADD) { d[i] = fma(d[i], a, b); n[i] = (n[i] ^ it) + 0x1234; }
            if (OP == FFMA_IADD) { f[i] = fmaf(f[i], fa, fb); n[i] = (n[i] ^ it) + 0x1234; }
            if (OP == DSETSEL) { d[i] = d[i] > b ? a : d[i] + 0.0 * b; }
            if (OP == DFMA_LDS) { d[i] = fma(d[i], a, sm[(n[i] + it) & 1023]); }
            if (OP == DFMA_D2F) { d[i] = fma(fma(fma(fma(d[i], a, b), a, b), a, b), a, b); f[i] += __double2float_rn(d[i]); }
            if (OP == DFMA_MUFU) { double y; d[i] = fma(fma(fma(fma(d[i], a, b), a, b), a, b), a, b); asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d[i])); d[i] = y; }
            if (OP == I2D) { d[i] = (double)n[i]; n[i] = __double2hiint(d[i]) + i; }
            if (OP == D2I) { n[i] = __double2int_rz(d[i]); d[i] = __hiloint2double(0x40000000 + (n[i] & 0xfffff), n[i]); }
            if (OP == DMNMX) d[i] = fmax(d[i] * a, b);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) s += d[i] + f[i] + n[i];
    if (s == 123456.789) out[0] = s;
}

template <int OP>
void run(double* out, int sms, double clk_ghz) {
    const int blocks = sms * 4, threads = 256, iters = 4000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
        cudaEventRecord(e0);
        k<OP><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (r && ms < best) best = ms;
    }
    int per = 1;
    if (OP == DFMA_D2F || OP == DFMA_MUFU) per = 5;
    if (OP == DFMA_FFMA || OP == DFMA_IADD || OP == FFMA_IADD || OP == DFMA_LDS) per = 2;
    if (OP == DMNMX) per = 2;
    double ops = (double)CHAINS * iters * blocks * threads;  // loop-body groups
    double groups_per_clk_sm = ops / (best * 1e-3) / (clk_ghz * 1e9) / sms;
    printf("%-18s %8.3f ms  %7.2f body-groups/clk/SM (%d instr of interest per group; excludes helper int ops)\n",
           NAMES[OP], best, groups_per_clk_sm, per);
}

__global__ void k_prec(const double* x, double* err, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double v = x[i], y, z;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(v));
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(z) : "d"(v));
    err[4 * i] = fabs(y * v - 1.0);
    err[4 * i + 1] = fabs(z * z * v - 1.0) * 0.5;
    double e = fma(-v, y, 1.0); double y1 = fma(y, e, y);
    err[4 * i + 2] = fabs(y1 - 1.0 / v) * v;
    double t = v * z; double e2 = fma(-t, z, 1.0); double z1 = fma(0.5 * z, e2, z);
    err[4 * i + 3] = fabs(z1 - 1.0 / sqrt(v)) * sqrt(v);
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double ghz = clk * 1e-6;
    printf("SMs %d, clock %.3f GHz (nominal max; rates below assume it)\n", sms, ghz);
    double* out; cudaMalloc(&out, 64);
    run<DFMA>(out, sms, ghz); run<DADD>(out, sms, ghz); run<DMUL>(out, sms, ghz); run<D2F>(out, sms, ghz);
    run<F2D>(out, sms, ghz); run<RCP64>(out, sms, ghz); run<RSQ64>(out, sms, ghz); run<F2I>(out, sms, ghz);
    run<FFMA>(out, sms, ghz); run<DFMA_FFMA>(out, sms, ghz); run<DFMA_IADD>(out, sms, ghz); run<FFMA_IADD>(out, sms, ghz);
    run<DSETSEL>(out, sms, ghz); run<DFMA_LDS>(out, sms, ghz); run<DFMA_D2F>(out, sms, ghz); run<DFMA_MUFU>(out, sms, ghz);
    run<I2D>(out, sms, ghz); run<D2I>(out, sms, ghz); run<DMNMX>(out, sms, ghz);
    const int n = 1 << 20;
    double* hx = (double*)malloc(n * sizeof(double));
    srand(1);
    for (int i = 0; i < n; ++i) hx[i] = ldexp(0.5 + 0.5 * rand() / (double)RAND_MAX + rand() * 1e-12, (rand() % 40) - 20);
    double *dx, *de; cudaMalloc(&dx, n * 8); cudaMalloc(&de, n * 32);
    cudaMemcpy(dx, hx, n * 8, cudaMemcpyHostToDevice);
    k_prec<<<n / 256, 256>>>(dx, de, n);
    double* he = (double*)malloc(n * 32);
    cudaMemcpy(he, de, n * 32, cudaMemcpyDeviceToHost);
    double m[4] = {0, 0, 0, 0};
    for (int i = 0; i < n; ++i) for (int j = 0; j < 4; ++j) if (he[4 * i + j] > m[j]) m[j] = he[4 * i + j];
    printf("max rel err: rcp seed %.3e (2^%.1f)  rsqrt seed %.3e (2^%.1f)  rcp+1 Newton %.3e  rsqrt+1 Newton %.3e\n",
           m[0], log2(m[0]), m[1], log2(m[1]), m[2], m[3]);
    return 0;
}
