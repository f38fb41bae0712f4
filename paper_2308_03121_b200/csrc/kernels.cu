// kernels.cu -- generic (LDG) conversion kernels of the NNVISR frame<->tensor
// path, sm_100a, and the launch dispatch between them and the TMA-pipelined
// kernels of kernels_tma.cu.
//
// f2t: frames -> NCHW tensor (steps A3-A7 of SURVEY.md §8(a); §3.1
//      P:282-304 pixel format / colourspace, §3.3 P:373-379 slot layout).
// t2f: NCHW tensor -> frames (steps B1-B4; north_star "RGB->YUV matrix,
//      chroma downsampling, scale, round-half-even and clamp").
//
// The generic kernels handle every geometry (odd widths, unaligned pitches,
// tensors whose rows are not 16-byte multiples): one thread converts one item
// of ROWS rows x 8 columns (ROWS = 2 for 4:2:0, the row pair sharing a chroma
// row; 1 otherwise) per grid-stride step, with 128-bit loads where aligned
// and a scalar path that clamps every coordinate elsewhere.  Frames of the
// common layouts go to the TMA-pipelined kernels instead (kernels_tma.cu).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace nnvisr {
namespace {
using namespace dev;

template <int FAMILY, typename IN, typename OUT>
__global__ void __launch_bounds__(kThreads) f2t_generic(const F2TArgs a)
{
    constexpr int ROWS = (FAMILY == kYUV420) ? 2 : 1;
    using V8 = typename Pack<IN>::V8;
    using V4 = typename Pack<IN>::V4;
    int cj = -1;
    DstList dl;
    DevFrame f;
    for (int64_t item = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; item < a.items;
         item += static_cast<int64_t>(gridDim.x) * kThreads) {
        const int job = static_cast<int>(item / a.units);
        const int unit = static_cast<int>(item - static_cast<int64_t>(job) * a.units);
        if (job != cj) {
            cj = job;
            f = load_frame(a.frames + a.job_frame[job]);
            dl.load(a, job);
        }
        const int ru = unit / a.col_units;
        const int x0 = (unit - ru * a.col_units) * kPx;
        const int y0 = ru * ROWS;
        const bool fast = a.vec_in && x0 + kPx <= a.W;
        Row8<OUT> out[ROWS][3];
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            const int yc = min(y0 + r, a.H - 1);
            int ys[kPx], us[kPx], vs[kPx];
            if (fast) {
                unpack8(*reinterpret_cast<const V8 *>(row_ptr<IN>(f, 0, yc) + x0), ys);
#pragma unroll
                for (int k = 0; k < kPx; ++k) ys[k] *= 16;
                if constexpr (FAMILY == kYUV420) {
                    const int cw = a.W >> 1, i0 = x0 >> 1;
                    const int rows[2] = {chroma_near(yc), chroma_far(yc, a.H >> 1)};
#pragma unroll
                    for (int p = 1; p <= 2; ++p) {
                        int h[2][kPx];
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            const IN *row = row_ptr<IN>(f, p, rows[q]);
                            int c[6];
                            unpack4(*reinterpret_cast<const V4 *>(row + i0), &c[1]);
                            c[0] = load1(row + max(i0 - 1, 0));
                            c[5] = load1(row + min(i0 + 4, cw - 1));
                            if (a.left) hup_left(c, h[q]);
                            else hup(c, h[q]);
                        }
#pragma unroll
                        for (int k = 0; k < kPx; ++k) {
                            const int s = 3 * h[0][k] + h[1][k];
                            if (p == 1) us[k] = s; else vs[k] = s;
                        }
                    }
                } else {
                    unpack8(*reinterpret_cast<const V8 *>(row_ptr<IN>(f, 1, yc) + x0), us);
                    unpack8(*reinterpret_cast<const V8 *>(row_ptr<IN>(f, 2, yc) + x0), vs);
#pragma unroll
                    for (int k = 0; k < kPx; ++k) {
                        us[k] *= 16;
                        vs[k] *= 16;
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < kPx; ++k)
                    f2t_codes_scalar<FAMILY, IN>(f, a.W, a.H, x0 + k, y0 + r, ys[k], us[k], vs[k], a.left);
            }
            f2t_row<FAMILY, OUT>(a.col, ys, us, vs, out[r]);
        }
        f2t_store<ROWS, OUT>(a, dl, out, x0, y0);
    }
}

// Left neighbour (column max(x0-1, 0)) of a row for LEFT siting: B-Y', R-Y'.
template <typename TIN, typename AR>
__device__ __forceinline__ void t2f_left_tap(const T2FConst<AR> &c, const TIN *row, int64_t plane, int x0, AR &lb,
                                             AR &lr)
{
    const int xl = max(x0 - 1, 0);
    const AR r_ = tload1(row + xl), g_ = tload1(row + plane + xl), b_ = tload1(row + 2 * plane + xl);
    const AR Y = fma_(c.kb, b_ - g_, fma_(c.kr, r_ - g_, g_));
    lb = b_ - Y;
    lr = r_ - Y;
}

template <int FAMILY, typename OS, typename TIN, typename AR, bool LEFT>
__device__ __forceinline__ void t2f_item(const T2FArgs &a, const T2FConst<AR> &c, const DevFrame &f, const TIN *src,
                                         int64_t plane, int x0, int y0)
{
    constexpr int ROWS = (FAMILY == kYUV420) ? 2 : 1;
    const int nvalid = min(kPx, a.Wo - x0);
    const bool vec_store = a.vec_out && nvalid == kPx;
    AR sb[4], sr[4];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        float R[kPx], G[kPx], B[kPx];
        const TIN *row = src + static_cast<int64_t>(r) * a.tw;
        if (a.vec_in && nvalid == kPx) {
            tload8_stream(row, R);
            tload8_stream(row + plane, G);
            tload8_stream(row + 2 * plane, B);
        } else {
#pragma unroll
            for (int k = 0; k < kPx; ++k) {
                const bool in = k < nvalid;
                R[k] = in ? tload1(row + k) : 0.f;
                G[k] = in ? tload1(row + plane + k) : 0.f;
                B[k] = in ? tload1(row + 2 * plane + k) : 0.f;
            }
        }
        AR lb = AR(0), lr = AR(0);
        if constexpr (LEFT) t2f_left_tap<TIN, AR>(c, row - x0, plane, x0, lb, lr);
        t2f_row<FAMILY, OS, AR, LEFT>(c, a.col, f, x0, y0 + r, r, R, G, B, nvalid, vec_store, sb, sr, lb, lr);
    }
    if constexpr (FAMILY == kYUV420) t2f_chroma420<OS, AR, LEFT>(c, f, x0, y0, sb, sr, nvalid, vec_store);
}

template <int FAMILY, typename OS, typename TIN, typename AR>
__global__ void __launch_bounds__(kThreads) t2f_generic(const T2FArgs a)
{
    constexpr int ROWS = (FAMILY == kYUV420) ? 2 : 1;
    const int64_t plane = a.th * a.tw;
    const T2FConst<AR> c(a.col);
    int cj = -1;
    DevFrame f;
    for (int64_t item = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; item < a.items;
         item += static_cast<int64_t>(gridDim.x) * kThreads) {
        const int job = static_cast<int>(item / a.units);
        const int unit = static_cast<int>(item - static_cast<int64_t>(job) * a.units);
        if (job != cj) {
            cj = job;
            f = load_frame(a.out + job);
        }
        const int ru = unit / a.col_units;
        const int x0 = (unit - ru * a.col_units) * kPx;
        const int y0 = ru * ROWS;
        int tup, o;
        t2f_job(a, job, tup, o);
        const TIN *src = reinterpret_cast<const TIN *>(a.src + static_cast<int64_t>(tup) * a.tensor_stride) +
                         static_cast<int64_t>(3 * o) * plane + static_cast<int64_t>(y0) * a.tw + x0;
        if (FAMILY == kYUV420 && a.left) t2f_item<FAMILY, OS, TIN, AR, true>(a, c, f, src, plane, x0, y0);
        else t2f_item<FAMILY, OS, TIN, AR, false>(a, c, f, src, plane, x0, y0);
    }
}

int sm_count()
{
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    return sms;
}

template <typename K, typename A>
cudaError_t launch_generic(K kernel, const A &a, cudaStream_t s)
{
    if (a.items <= 0) return cudaSuccess;
    const int64_t tiles = (a.items + kThreads - 1) / kThreads;
    const int grid = static_cast<int>(std::min<int64_t>(tiles, static_cast<int64_t>(sm_count()) * 16));
    kernel<<<grid, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

template <int FAMILY>
cudaError_t f2t_dispatch(int bits, int dtype, const F2TArgs &a, cudaStream_t s)
{
    if (bits == 8) {
        if (dtype == kF16) return launch_generic(f2t_generic<FAMILY, uint8_t, __half>, a, s);
        return launch_generic(f2t_generic<FAMILY, uint8_t, float>, a, s);
    }
    if (dtype == kF16) return launch_generic(f2t_generic<FAMILY, uint16_t, __half>, a, s);
    return launch_generic(f2t_generic<FAMILY, uint16_t, float>, a, s);
}

template <int FAMILY>
cudaError_t t2f_dispatch(int bits, int dtype, const T2FArgs &a, cudaStream_t s)
{
    if (bits == 8) {
        if (dtype == kF16) return launch_generic(t2f_generic<FAMILY, uint8_t, __half, float>, a, s);
        return launch_generic(t2f_generic<FAMILY, uint8_t, float, float>, a, s);
    }
    if (bits == 10) {
        if (dtype == kF16) return launch_generic(t2f_generic<FAMILY, uint16_t, __half, float>, a, s);
        return launch_generic(t2f_generic<FAMILY, uint16_t, float, float>, a, s);
    }
    // 16-bit codes: fp32 arithmetic leaves ~0.2% of codes 1 LSB off the exact
    // result, so B2/B4 run in fp64 (SURVEY.md §7 "Numerics at 16-bit").
    if (dtype == kF16) return launch_generic(t2f_generic<FAMILY, uint16_t, __half, double>, a, s);
    return launch_generic(t2f_generic<FAMILY, uint16_t, float, double>, a, s);
}

}  // namespace

cudaError_t launch_f2t(int family, int bits, int dtype, const F2TArgs &a, cudaStream_t s)
{
    count_launch();
    if (a.yuv) return launch_f2t_yuv(family, bits, dtype, a, s);
    if (a.tma_ok) {
        // low fan-out 4:2:0 launches (each converted frame written to < 1.5
        // slots on average: store mode, Fig. 1 slots) are bound by the
        // conversion, not HBM: the lean row-marching kernel (kernels_strip.cu;
        // B200: c2 store 5.2 vs 4.1 TB/s, c4 batches 4.2 vs 3.8; 2-frame
        // windows stay on the TMA pipeline, 5.3 vs 4.9);
        // NNVISR_F2T_STRIP = 0 / 1 forces the choice (A/B experiments)
        const char *e = std::getenv("NNVISR_F2T_STRIP");
        const int force = e && *e ? std::atoi(e) : -1;
        const bool low = 2 * a.dests < 3 * a.jobs;
        if (family == kYUV420 && f2t_strip_ok(dtype, a) && (force == 1 || (force < 0 && low)))
            return launch_f2t_strip(bits, dtype, a, s);
        return launch_f2t_tma(family, bits, dtype, a, s);
    }
    switch (family) {
    case kYUV420: return f2t_dispatch<kYUV420>(bits, dtype, a, s);
    case kYUV444: return f2t_dispatch<kYUV444>(bits, dtype, a, s);
    default: return f2t_dispatch<kRGB>(bits, dtype, a, s);
    }
}

cudaError_t launch_t2f(int family, int bits, int dtype, const T2FArgs &a, cudaStream_t s)
{
    count_launch();
    if (a.yuv) return launch_t2f_yuv(family, bits, dtype, a, s);
    if (a.tma_ok) return launch_t2f_tma(family, bits, dtype, a, s);
    switch (family) {
    case kYUV420: return t2f_dispatch<kYUV420>(bits, dtype, a, s);
    case kYUV444: return t2f_dispatch<kYUV444>(bits, dtype, a, s);
    default: return t2f_dispatch<kRGB>(bits, dtype, a, s);
    }
}

}  // namespace nnvisr
