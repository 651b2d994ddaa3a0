// Output packing (outputs.py) and evaluation metrics (metrics.py) of the reference, on the
// device: the rows SURVEY.md section 8(f) ranks next after the hot path (f3, f4).  All of it is
// HBM-bound byte / index work: one pass over the points or pixels, no reuse.
//
// Reference shorthand: O = pkg/src/densify360/outputs.py, M = pkg/src/densify360/metrics.py.
#include <math.h>

#include "d360_device.cuh"

namespace d360 {

static inline unsigned io_blocks(size_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

// O:30-54: record = astype(float32) of (x, y, z), little endian, then r, g, b (15 bytes, packed).
// A block packs 256 records into shared memory and writes them out as 240 aligned 16-byte
// stores (a record-per-thread byte store pattern runs at a sixth of the HBM rate).
constexpr int PLY_BLOCK = 256;
__global__ void __launch_bounds__(PLY_BLOCK)
    k_pack_ply(const double* __restrict__ pts, const uint8_t* __restrict__ rgb, uint8_t* __restrict__ rec, size_t n) {
    __shared__ __align__(16) uint8_t sh[PLY_BLOCK * 15];
    const size_t base = (size_t)blockIdx.x * PLY_BLOCK;
    const size_t i = base + threadIdx.x;
    if (i < n) {
        uint8_t* o = sh + 15 * threadIdx.x;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const unsigned b = __float_as_uint(__double2float_rn(pts[3 * i + c]));
            o[4 * c + 0] = (uint8_t)(b);
            o[4 * c + 1] = (uint8_t)(b >> 8);
            o[4 * c + 2] = (uint8_t)(b >> 16);
            o[4 * c + 3] = (uint8_t)(b >> 24);
        }
        o[12] = rgb[3 * i];
        o[13] = rgb[3 * i + 1];
        o[14] = rgb[3 * i + 2];
    }
    __syncthreads();
    const size_t n_here = n - base < (size_t)PLY_BLOCK ? n - base : (size_t)PLY_BLOCK;
    const size_t bytes = n_here * 15;
    uint8_t* out = rec + base * 15;  // 3840 * blockIdx: 16-byte aligned when rec is
    const size_t vec = ((reinterpret_cast<uintptr_t>(out) & 15) == 0) ? bytes / 16 : 0;
    for (size_t k = threadIdx.x; k < vec; k += PLY_BLOCK)
        reinterpret_cast<uint4*>(out)[k] = reinterpret_cast<const uint4*>(sh)[k];
    for (size_t k = vec * 16 + threadIdx.x; k < bytes; k += PLY_BLOCK) out[k] = sh[k];
}

// order-preserving map f32 -> u32 (for atomicMin / atomicMax on depths of any sign)
__device__ __forceinline__ unsigned f32_key(float f) {
    const unsigned b = __float_as_uint(f);
    return b ^ ((b >> 31) ? 0xffffffffu : 0x80000000u);
}

__global__ void k_mm16_init(unsigned* stats) {
    stats[0] = 0u;           // valid count
    stats[1] = 0xffffffffu;  // min key
    stats[2] = 0u;           // max key
}

// O:81-97: mm = clip(rint(depth * 1000), 0, 65535) computed in f64, 0 where invalid; the sidecar's
// valid count and min / max valid depth come out of the same pass (grid-stride, one set of
// atomics per block).
constexpr int MM_THREADS = 256;
__global__ void __launch_bounds__(MM_THREADS)
    k_depth_to_mm16(const float* __restrict__ depth, const uint8_t* __restrict__ valid, uint16_t* __restrict__ mm,
                    unsigned* stats, size_t n) {
    unsigned cnt = 0, kmin = 0xffffffffu, kmax = 0u;
    for (size_t i = (size_t)blockIdx.x * MM_THREADS + threadIdx.x; i < n; i += (size_t)gridDim.x * MM_THREADS) {
        const float d = depth[i];
        double v = rint((double)d * 1000.0);  // np.rint: half to even
        v = v < 0.0 ? 0.0 : (v > 65535.0 ? 65535.0 : v);
        const bool ok = valid[i] != 0;
        mm[i] = ok ? (uint16_t)v : (uint16_t)0;
        if (ok) {
            const unsigned k = f32_key(d);
            ++cnt;
            kmin = min(kmin, k);
            kmax = max(kmax, k);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    __shared__ unsigned sh[3][MM_THREADS / 32];
    if ((threadIdx.x & 31) == 0) {
        sh[0][threadIdx.x >> 5] = cnt;
        sh[1][threadIdx.x >> 5] = kmin;
        sh[2][threadIdx.x >> 5] = kmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < MM_THREADS / 32; ++w) {
            cnt += sh[0][w];
            kmin = min(kmin, sh[1][w]);
            kmax = max(kmax, sh[2][w]);
        }
        if (cnt) {
            atomicAdd(&stats[0], cnt);
            atomicMin(&stats[1], kmin);
            atomicMax(&stats[2], kmax);
        }
    }
}

struct PoseDev {
    double r[9], t[3];
};

// M:31-43: local = (p - t) @ R; points at the camera centre dropped; nearest pixel by np.rint
// (half to even), columns modulo W, rows clipped.  Marks the raster (idempotent byte stores).
__global__ void k_completeness_splat(const double* __restrict__ pts, size_t n, const __grid_constant__ PoseDev pose,
                                     uint8_t* __restrict__ raster, int H, int W) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double dx = pts[3 * i] - pose.t[0], dy = pts[3 * i + 1] - pose.t[1], dz = pts[3 * i + 2] - pose.t[2];
    const double* R = pose.r;
    const double lx = __dadd_rn(__dadd_rn(__dmul_rn(dx, R[0]), __dmul_rn(dy, R[3])), __dmul_rn(dz, R[6]));
    const double ly = __dadd_rn(__dadd_rn(__dmul_rn(dx, R[1]), __dmul_rn(dy, R[4])), __dmul_rn(dz, R[7]));
    const double lz = __dadd_rn(__dadd_rn(__dmul_rn(dx, R[2]), __dmul_rn(dy, R[5])), __dmul_rn(dz, R[8]));
    const double r = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(lx, lx), __dmul_rn(ly, ly)), __dmul_rn(lz, lz)));
    if (!(r > 1e-12)) return;
    double lon = atan2(lx, lz);
    if (lon >= D360_PI) lon -= 2.0 * D360_PI;
    const double u = (lon + D360_PI) * ((double)W / (2.0 * D360_PI)) - 0.5;
    double s = -ly / r;
    s = s < -1.0 ? -1.0 : (s > 1.0 ? 1.0 : s);
    const double v = acos(s) * ((double)H / D360_PI) - 0.5;
    long long px = (long long)rint(u) % W;
    if (px < 0) px += W;
    long long py = (long long)rint(v);
    py = py < 0 ? 0 : (py > H - 1 ? H - 1 : py);
    raster[(size_t)py * W + px] = 1;
}

__global__ void k_count_nonzero(const uint8_t* __restrict__ a, size_t n, unsigned long long* count) {
    unsigned c = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        c += a[i] != 0;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, (unsigned long long)c);
}

// M:52-78 over jointly valid pixels: sum |p - g| / g, sum (p - g)^2, #(rel <= 0.02), #joint.
// Two stages with a fixed reduction order, so the f64 sums are the same on every run.
constexpr int ACC_BLOCKS = 1024, ACC_THREADS = 256;
__global__ void __launch_bounds__(ACC_THREADS)
    k_accuracy_partial(const float* __restrict__ pd, const uint8_t* __restrict__ pv, const float* __restrict__ gd,
                       const uint8_t* __restrict__ gv, size_t n, double* __restrict__ partial) {
    __shared__ double sh[4][ACC_THREADS];
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    for (size_t i = (size_t)blockIdx.x * ACC_THREADS + threadIdx.x; i < n; i += (size_t)ACC_BLOCKS * ACC_THREADS) {
        if (pv[i] && gv[i]) {
            const double p = (double)pd[i], g = (double)gd[i];
            const double rel = fabs(p - g) / g;
            a[0] += rel;
            a[1] += (p - g) * (p - g);
            a[2] += rel <= 0.02 ? 1.0 : 0.0;
            a[3] += 1.0;
        }
    }
    for (int k = 0; k < 4; ++k) sh[k][threadIdx.x] = a[k];
    __syncthreads();
    for (int o = ACC_THREADS / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            for (int k = 0; k < 4; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x < 4) partial[threadIdx.x * ACC_BLOCKS + blockIdx.x] = sh[threadIdx.x][0];
}
__global__ void __launch_bounds__(ACC_BLOCKS) k_accuracy_final(const double* __restrict__ partial, double* out) {
    __shared__ double sh[4][ACC_BLOCKS];
    for (int k = 0; k < 4; ++k) sh[k][threadIdx.x] = partial[k * ACC_BLOCKS + threadIdx.x];
    __syncthreads();
    for (int o = ACC_BLOCKS / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            for (int k = 0; k < 4; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x < 4) out[threadIdx.x] = sh[threadIdx.x][0];
}

// M:81-87: cell = floor(p / voxel) per axis, packed 21 bits each into one sortable key
__global__ void k_voxel_keys(const double* __restrict__ pts, size_t n, double voxel, long long* __restrict__ keys,
                             int* overflow) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    long long key = 0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const long long cell = (long long)floor(pts[3 * i + c] / voxel) + (1ll << 20);
        if (cell < 0 || cell >= (1ll << 21)) *overflow = 1;
        key = (key << 21) | (cell & ((1ll << 21) - 1));
    }
    keys[i] = key;
}

// ---------------------------------------------------------------------------------------
// Image ingest: dataset.resample_keyframe (reference dataset.py:146-157) = Pillow's
// Image.resize(..., LANCZOS) on 8-bit images.  Pillow is a third-party dependency absent from
// /root/reference (pinned: Pillow 12.2.0 in this image); its published algorithm
// (src/libImaging/Resample.c) is two separable passes - horizontal first, into a uint8
// intermediate, then vertical - each a convolution with per-output-pixel windows [xmin, xmin + n)
// and coefficients normalised and rounded to 22-bit fixed point; the accumulator starts at
// 1 << 21 (round half up) and the result is (acc >> 22) clipped to [0, 255].  The windows and the
// integer coefficients are computed on the host (ingest.py, Pillow's double arithmetic statement by
// statement: a few hundred values), the byte work runs here: pure integer, so bit-exact.
// HBM-bound: one read of the source, one write + read of the intermediate, one write.
// ---------------------------------------------------------------------------------------
constexpr int RESAMPLE_BITS = 22;

__device__ __forceinline__ uint8_t clip8_fixed(int v) {
    v >>= RESAMPLE_BITS;
    return (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v));
}

// One thread per output pixel, all channels.  horizontal: out (rows, out_w, C) from in rows [row0, row0 + rows)
// of (in_h, in_w, C); vertical: out (out_h, w, C) from in (in_h, w, C).
template <int C, bool VERTICAL>
__global__ void k_resample(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, const int* __restrict__ bounds,
                           const int* __restrict__ kk, int ksize, int in_w, int row0, int out_w, int out_h) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= out_w || y >= out_h) return;
    const int o = VERTICAL ? y : x;
    const int lo = __ldg(bounds + 2 * o), n = __ldg(bounds + 2 * o + 1);
    const int* k = kk + (size_t)o * ksize;
    int acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = 1 << (RESAMPLE_BITS - 1);
    for (int t = 0; t < n; ++t) {
        const size_t src = VERTICAL ? ((size_t)(lo + t) * out_w + x) * C : ((size_t)(y + row0) * in_w + lo + t) * C;
        const int w = __ldg(k + t);
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c] += (int)__ldg(in + src + c) * w;
    }
    const size_t dst = ((size_t)y * out_w + x) * C;
#pragma unroll
    for (int c = 0; c < C; ++c) out[dst + c] = clip8_fixed(acc[c]);
}

}  // namespace d360

using namespace d360;

extern "C" int d360_pack_ply_records(const double* points, const uint8_t* colors, uint8_t* records, int64_t n,
                                     void* stream) {
    if (n < 0) {
        set_error("pack_ply_records: n = %lld", (long long)n);
        return 1;
    }
    if (n == 0) return 0;
    {
        TraceScope ts_("pack_ply", (cudaStream_t)stream);
        k_pack_ply<<<io_blocks((size_t)n, PLY_BLOCK), PLY_BLOCK, 0, (cudaStream_t)stream>>>(points, colors, records, (size_t)n);
    }
    return check_launch("pack_ply_records");
}

extern "C" int d360_depth_to_mm16(const float* depth, const uint8_t* valid, uint16_t* mm, uint32_t* stats, int height,
                                  int width, void* stream) {
    const size_t n = (size_t)height * width;
    {
        TraceScope ts_("depth_to_mm16", (cudaStream_t)stream);
        k_mm16_init<<<1, 1, 0, (cudaStream_t)stream>>>(stats);
        k_depth_to_mm16<<<min(io_blocks(n, MM_THREADS), 148u * 8u), MM_THREADS, 0, (cudaStream_t)stream>>>(depth, valid, mm, stats, n);
    }
    return check_launch("depth_to_mm16");
}

extern "C" int d360_completeness_splat(const double* points, int64_t n, const double* rot, const double* trans,
                                       uint8_t* raster, int height, int width, void* stream) {
    if (n <= 0) return 0;
    PoseDev pose;
    for (int i = 0; i < 9; ++i) pose.r[i] = rot[i];
    for (int i = 0; i < 3; ++i) pose.t[i] = trans[i];
    {
        TraceScope ts_("completeness_splat", (cudaStream_t)stream);
        k_completeness_splat<<<io_blocks((size_t)n, 256), 256, 0, (cudaStream_t)stream>>>(points, (size_t)n, pose, raster,
                                                                                        height, width);
    }
    return check_launch("completeness_splat");
}

extern "C" int d360_count_nonzero(const uint8_t* a, int64_t n, unsigned long long* count, void* stream) {
    if (n <= 0) return 0;
    {
        TraceScope ts_("count_nonzero", (cudaStream_t)stream);
        k_count_nonzero<<<min(io_blocks((size_t)n, 256), 1184u), 256, 0, (cudaStream_t)stream>>>(a, (size_t)n, count);
    }
    return check_launch("count_nonzero");
}

extern "C" int d360_accuracy_scratch_doubles(void) { return 4 * ACC_BLOCKS; }

extern "C" int d360_depth_accuracy(const float* pred_depth, const uint8_t* pred_valid, const float* gt_depth,
                                   const uint8_t* gt_valid, int64_t n, double* scratch, double* out, void* stream) {
    {
        TraceScope ts_("depth_accuracy", (cudaStream_t)stream);
        k_accuracy_partial<<<ACC_BLOCKS, ACC_THREADS, 0, (cudaStream_t)stream>>>(pred_depth, pred_valid, gt_depth, gt_valid,
                                                                                (size_t)(n < 0 ? 0 : n), scratch);
        k_accuracy_final<<<1, ACC_BLOCKS, 0, (cudaStream_t)stream>>>(scratch, out);
    }
    return check_launch("depth_accuracy");
}

extern "C" int d360_voxel_keys(const double* points, int64_t n, double voxel, long long* keys, int* overflow,
                               void* stream) {
    if (!(voxel > 0.0)) {
        set_error("voxel edge must be > 0, got %g", voxel);
        return 1;
    }
    if (n <= 0) return 0;
    {
        TraceScope ts_("voxel_keys", (cudaStream_t)stream);
        k_voxel_keys<<<io_blocks((size_t)n, 256), 256, 0, (cudaStream_t)stream>>>(points, (size_t)n, voxel, keys, overflow);
    }
    return check_launch("voxel_keys");
}

extern "C" int d360_resample_u8(const uint8_t* src, int src_h, int src_w, int channels, uint8_t* tmp, uint8_t* dst,
                                int dst_h, int dst_w, const int32_t* bounds_x, const int32_t* kk_x, int ksize_x,
                                const int32_t* bounds_y, const int32_t* kk_y, int ksize_y, int row0, int rows,
                                void* stream) {
    if (channels != 1 && channels != 3) {
        set_error("resample: expected 1 or 3 channels, got %d", channels);
        return 1;
    }
    if (src_h < 1 || src_w < 1 || dst_h < 1 || dst_w < 1 || ksize_x < 1 || ksize_y < 1 || row0 < 0 || rows < 1 ||
        row0 + rows > src_h) {
        set_error("resample: bad sizes (src %dx%d, dst %dx%d, rows [%d, %d))", src_w, src_h, dst_w, dst_h, row0,
                  row0 + rows);
        return 1;
    }
    cudaStream_t s = (cudaStream_t)stream;
    {   // horizontal pass over the source rows the vertical pass will read (Resample.c: ybox_first .. ybox_last)
        dim3 grid((dst_w + 127) / 128, rows);
        TraceScope ts_("resample_h", s);
        if (channels == 3) k_resample<3, false><<<grid, 128, 0, s>>>(src, tmp, bounds_x, kk_x, ksize_x, src_w, row0, dst_w, rows);
        else k_resample<1, false><<<grid, 128, 0, s>>>(src, tmp, bounds_x, kk_x, ksize_x, src_w, row0, dst_w, rows);
    }
    if (check_launch("resample/horizontal")) return 2;
    {
        dim3 grid((dst_w + 127) / 128, dst_h);
        TraceScope ts_("resample_v", s);
        if (channels == 3) k_resample<3, true><<<grid, 128, 0, s>>>(tmp, dst, bounds_y, kk_y, ksize_y, dst_w, 0, dst_w, dst_h);
        else k_resample<1, true><<<grid, 128, 0, s>>>(tmp, dst, bounds_y, kk_y, ksize_y, dst_w, 0, dst_w, dst_h);
    }
    return check_launch("resample/vertical");
}
