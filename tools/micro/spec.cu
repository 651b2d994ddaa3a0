// Does warp specialisation beat a homogeneous instruction mix on the issue port / FP64 pipe?
// 16 warps per SM (4 per scheduler).  Work per "unit": ND D-ops + NF FFMA + NS SHF (the cost kernels' mix is
// roughly 51 : 25 : 20 per sample-view).  homogeneous: every warp runs units of the full mix;
// specialised: 3 of 4 warps per scheduler run the FP64-heavy part, 1 of 4 runs the rest of 3 units.
// nvcc -O3 -arch=sm_100a spec.cu -o spec   (experiment, not part of the product)
#include <cstdio>
#include <cuda_runtime.h>

template <int ND, int NF, int NS>
__device__ __forceinline__ void unit(double (&d)[8], float (&f)[8], unsigned (&n)[8], double a, double b, float fa) {
#pragma unroll
    for (int j = 0; j < ND; ++j) d[j & 7] = fma(d[j & 7], a, b);
#pragma unroll
    for (int j = 0; j < NF; ++j) f[j & 7] = fmaf(f[j & 7], fa, 1e-3f);
#pragma unroll
    for (int j = 0; j < NS; ++j) n[j & 7] = __funnelshift_l(n[j & 7], n[j & 7], 3 + (j & 3));
}

// MODE 0: homogeneous (ND, NF, NS per unit, `units` units per warp)
// MODE 1: specialised: warps 0..11: (PD, PF, PS) per unit; warps 12..15: 3 x (CD, CF, CS) per unit
template <int MODE, int ND, int NF, int NS, int PD, int PF, int PS>
__global__ void __launch_bounds__(512, 1) k(double* out, long long* cyc, int units, double a, double b, float fa) {
    double d[8]; float f[8]; unsigned n[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { d[i] = a + threadIdx.x * 1e-3 + i; f[i] = (float)d[i]; n[i] = threadIdx.x * 7 + i; }
    __syncthreads();
    long long t0 = clock64();
    const int warp = threadIdx.x >> 5;
    if (MODE == 0) {
        for (int u = 0; u < units; ++u) unit<ND, NF, NS>(d, f, n, a, b, fa);
    } else if (warp < 12) {
        for (int u = 0; u < units; ++u) unit<PD, PF, PS>(d, f, n, a, b, fa);
    } else {
        for (int u = 0; u < units; ++u) {
            unit<ND - PD, NF - PF, NS - PS>(d, f, n, a, b, fa);
            unit<ND - PD, NF - PF, NS - PS>(d, f, n, a, b, fa);
            unit<ND - PD, NF - PF, NS - PS>(d, f, n, a, b, fa);
        }
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += d[i] + f[i] + n[i];
    if (s == 123456.789) out[0] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int MODE, int ND, int NF, int NS, int PD, int PF, int PS>
void run(const char* name, double* out, long long* cyc) {
    const int units = 400;
    // homogeneous: 16 warps x units; specialised: 12 producer warps x units (+ 4 consumer warps doing the rest of 3 units each):
    // to compare equal total work, the homogeneous run does units * 12 / 16
    const int u = MODE == 0 ? units * 12 / 16 : units;
    k<MODE, ND, NF, NS, PD, PF, PS><<<1, 512>>>(out, cyc, u, 1.0000001, 1e-9, 1.0001f);
    k<MODE, ND, NF, NS, PD, PF, PS><<<1, 512>>>(out, cyc, u, 1.0000001, 1e-9, 1.0001f);
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    // total units of full mix processed per scheduler = units * 3 (12 warps / 4 schedulers)
    printf("%-40s %.1f clk per unit per scheduler (FP64 floor %.1f, issue floor %.1f)\n", name, (double)h / (units * 3.0),
           ND * 2.04, ND * 1.5 + NF + NS);
}
int main() {
    double* out; long long* cyc; cudaMalloc(&out, 64); cudaMalloc(&cyc, 8);
    run<0, 51, 27, 20, 0, 0, 0>("homogeneous 51 D + 27 F + 20 S", out, cyc);
    run<1, 51, 27, 20, 44, 10, 10>("specialised P(44,10,10) C(7,17,10)", out, cyc);
    run<1, 51, 27, 20, 51, 0, 0>("specialised P(51,0,0) C(0,27,20)", out, cyc);
    run<0, 51, 17, 12, 0, 0, 0>("homogeneous 51 D + 17 F + 12 S", out, cyc);
    run<1, 51, 17, 12, 44, 6, 6>("specialised P(44,6,6) C(7,11,6)", out, cyc);
    return 0;
}
