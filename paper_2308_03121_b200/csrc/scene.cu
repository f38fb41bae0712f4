// scene.cu -- scene-change detection (SPEC.md
// scenedetect.detect_scene_changes): per consecutive frame pair the exact
// integer sum of absolute luma differences, then the threshold decision on
// the normalised mean.  A read-only streaming pass over the luma planes
// (HBM-bound; a block walks 8 consecutive frames row by row, so each frame
// row is read from memory once).
#include <algorithm>

#include "common.cuh"

namespace nnvisr {
namespace {
using namespace dev;

constexpr int kSadRowsPerBlock = 8;

template <typename IN>
__device__ __forceinline__ int luma_at(const DevFrame &f, int x, int y, bool rgb)
{
    if (!rgb) return load1(row_ptr<IN>(f, 0, y) + x);
    return 299 * load1(row_ptr<IN>(f, 0, y) + x) + 587 * load1(row_ptr<IN>(f, 1, y) + x) +
           114 * load1(row_ptr<IN>(f, 2, y) + x);
}

constexpr int kSadFrames = 8;  // consecutive frames per block: each frame row is read once

// grid: (row blocks, frame groups).  Block (rows [blockIdx.x * R, ...),
// frames first = blockIdx.y * kSadFrames .. first + kSadFrames, clamped): for
// every row, thread t walks its 8-column groups through the group's frames,
// keeping the previous frame's samples in registers, so every frame row is
// read from memory once (plus the group's first frame, shared with the
// previous group).
template <typename IN>
__global__ void __launch_bounds__(kThreads, 4) sad_kernel(const DevFrame *frames, int count, int W, int H, int vec,
                                                       int rgb, unsigned long long *sad)
{
    using V8 = typename Pack<IN>::V8;
    const int f0 = blockIdx.y * kSadFrames;
    const int nf = min(kSadFrames, count - 1 - f0);  // pairs (f0+j, f0+j+1), j < nf
    if (nf <= 0) return;
    const int y0 = blockIdx.x * kSadRowsPerBlock, y1 = min(y0 + kSadRowsPerBlock, H);
    const int groups = (W + kPx - 1) / kPx;
    // per-thread sums fit 32 bits (<= 8 rows x 8 columns x 65535 per column group pass)
    unsigned long long acc[kSadFrames];
#pragma unroll
    for (int j = 0; j < kSadFrames; ++j) acc[j] = 0;
    if (vec && !rgb) {
        // one (row, 8-column group): all kSadFrames + 1 rows' loads first
        // (independent, in flight together; frames past the group's end
        // re-read its last one), then the differences
        auto item = [&](int y, int g) {
            const int x = g * kPx;
            if (x + kPx > W) return;
            V8 q[kSadFrames + 1];
#pragma unroll
            for (int j = 0; j <= kSadFrames; ++j)
                q[j] = *reinterpret_cast<const V8 *>(row_ptr<IN>(load_frame(frames + f0 + min(j, nf)), 0, y) + x);
            int prev[kPx];
            unpack8(q[0], prev);
#pragma unroll
            for (int j = 0; j < kSadFrames; ++j) {
                int cur[kPx];
                unpack8(q[j + 1], cur);
                uint32_t d = 0;
#pragma unroll
                for (int k = 0; k < kPx; ++k) {
                    d += static_cast<uint32_t>(abs(cur[k] - prev[k]));
                    prev[k] = cur[k];
                }
                acc[j] += d;
            }
        };
        if (groups < (3 * kThreads) / 4) {
            // narrow frames: (row, group) items over all the block's rows, so
            // every thread has work
            const int items = (y1 - y0) * groups;
            for (int it = threadIdx.x; it < items; it += kThreads) item(y0 + it / groups, it % groups);
        } else {
            for (int y = y0; y < y1; ++y)
                for (int g = threadIdx.x; g < groups; g += kThreads) item(y, g);
        }
    } else {
        for (int y = y0; y < y1; ++y) {
            for (int x = threadIdx.x; x < W; x += kThreads) {
                int prev = luma_at<IN>(load_frame(frames + f0), x, y, rgb);
                for (int j = 0; j < nf; ++j) {
                    const int cur = luma_at<IN>(load_frame(frames + f0 + j + 1), x, y, rgb);
                    acc[j] += static_cast<unsigned long long>(abs(cur - prev));
                    prev = cur;
                }
            }
        }
    }
    // block reduction per pair
    __shared__ unsigned long long part[kThreads / 32][kSadFrames];
#pragma unroll
    for (int j = 0; j < kSadFrames; ++j) {
        unsigned long long v = acc[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5][j] = v;
    }
    __syncthreads();
    if (threadIdx.x < nf) {
        unsigned long long v = 0;
        for (int w = 0; w < kThreads / 32; ++w) v += part[w][threadIdx.x];
        atomicAdd(sad + f0 + threadIdx.x + 1, v);
    }
}

__global__ void cut_kernel(const unsigned long long *sad, int count, double denom, double threshold, uint8_t *cut)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) cut[i] = static_cast<uint8_t>(i > 0 && static_cast<double>(sad[i]) / denom > threshold);
}

}  // namespace

cudaError_t launch_scene_detect(int family, int bits, int range, int W, int H, const DevFrame *frames, int count,
                                int vec, double threshold, uint64_t *sad, uint8_t *cut, cudaStream_t s)
{
    cudaError_t e = cudaMemsetAsync(sad, 0, sizeof(uint64_t) * count, s);
    if (e != cudaSuccess) return e;
    const bool rgb = family == kRGB;
    if (count > 1) {
        count_launch();
        const dim3 grid((H + kSadRowsPerBlock - 1) / kSadRowsPerBlock, (count - 1 + kSadFrames - 1) / kSadFrames);
        auto *out = reinterpret_cast<unsigned long long *>(sad);
        if (bits == 8) sad_kernel<uint8_t><<<grid, kThreads, 0, s>>>(frames, count, W, H, vec, rgb, out);
        else sad_kernel<uint16_t><<<grid, kThreads, 0, s>>>(frames, count, W, H, vec, rgb, out);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    // one code step of normalised luma (reading A2), x1000 for RGB luma
    double scale = range == 0 ? 219.0 * std::ldexp(1.0, bits - 8) : std::ldexp(1.0, bits) - 1.0;
    if (rgb) scale *= 1000.0;
    count_launch();
    cut_kernel<<<(count + 255) / 256, 256, 0, s>>>(reinterpret_cast<const unsigned long long *>(sad), count,
                                                   static_cast<double>(W) * H * scale, threshold, cut);
    return cudaGetLastError();
}

}  // namespace nnvisr
