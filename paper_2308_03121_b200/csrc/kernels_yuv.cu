// kernels_yuv.cu -- YUV-native network tensors (
// PAPER.md §3.1: "NNVISR supports input and output in both RGB and
// YUV pixel format ... YUV420 halves the spatial dimension of 2 in 3 of its
// channels").  The network sees the clip's own planes: no matrix and no
// chroma resampling, only the range (de)quantisation of readings A2-A4 with
// the chroma offset of reading A22 (U = Pb + 1/2).
//
// f2t: a job is one distinct frame; an item is ROWS luma rows x 8 columns
//      (ROWS = 2 for 4:2:0) plus the matching chroma row x 4 (4:2:0) or 8
//      columns of U and V, stored to every (run, slot) destination of the
//      frame.  Luma and chroma tensors are separate address streams
//      (F2TArgs::dst / dst2), padded per plane by edge replication.
// t2f: an item is ROWS output rows x 8 columns of luma plus the chroma row
//      x 4 (or 8) columns; B4 (scale, RNE, clamp) only.
//
// Both directions are pure streaming (each input byte read once, each output
// byte written once), so a grid-stride loop with 16-byte accesses where the
// geometry allows is the whole design; HBM bandwidth is the roofline.
#include <algorithm>

#include "common.cuh"

namespace nnvisr {
namespace {
using namespace dev;

template <int NC> struct RowN;
template <> struct RowN<4> { template <typename OUT> using T = Row4<OUT>; };
template <> struct RowN<8> { template <typename OUT> using T = Row8<OUT>; };

// NC samples of a row starting at x (vector load when `fast`, else clamped
// scalar loads against the plane width w)
template <typename IN, int NC>
__device__ __forceinline__ void load_codes(const IN *row, int x, int w, bool fast, int (&c)[NC])
{
    using V8 = typename Pack<IN>::V8;
    using V4 = typename Pack<IN>::V4;
    if (fast) {
        if constexpr (NC == 8) unpack8(*reinterpret_cast<const V8 *>(row + x), c);
        else unpack4(*reinterpret_cast<const V4 *>(row + x), c);
    } else {
#pragma unroll
        for (int k = 0; k < NC; ++k) c[k] = load1(row + min(x + k, w - 1));
    }
}

template <int FAMILY, typename IN, typename OUT>
__global__ void __launch_bounds__(kThreads) f2t_yuv_generic(const F2TArgs a)
{
    constexpr bool SUB = FAMILY == kYUV420;
    constexpr int ROWS = SUB ? 2 : 1, NC = SUB ? 4 : 8;
    using RowC = typename RowN<NC>::template T<OUT>;
    const int cw = SUB ? a.W >> 1 : a.W, ch = SUB ? a.H >> 1 : a.H;
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
        // luma: Y' = (16 c - y_off) * y_scale  (reading A2)
        Row8<OUT> ly[ROWS];
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            int c[kPx];
            load_codes<IN, kPx>(row_ptr<IN>(f, 0, min(y0 + r, a.H - 1)), x0, a.W, fast, c);
            float v[kPx];
#pragma unroll
            for (int k = 0; k < kPx; ++k) v[k] = static_cast<float>(16 * c[k] - a.col.y_off) * a.col.y_scale;
            ly[r].set(v);
        }
        // chroma: U = P + 1/2 = (16 c - u_off) * c_scale, u_off = c_off - 1/(2 c_scale)
        // an exact integer, so one rounding as for luma (reading A22)
        const int cy = SUB ? ru : y0, cx0 = SUB ? x0 >> 1 : x0;
        RowC lc[2];
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            int c[NC];
            load_codes<IN, NC>(row_ptr<IN>(f, 1 + p, min(cy, ch - 1)), cx0, cw, fast, c);
            float v[NC];
#pragma unroll
            for (int k = 0; k < NC; ++k) v[k] = static_cast<float>(16 * c[k] - a.col.u_off) * a.col.c_scale;
            lc[p].set(v);
        }
        const bool vl = a.vec_out && x0 + kPx <= a.Wp;
        const int nl = min(kPx, a.Wp - x0);
        const bool vc = a.vec_out_c && cx0 + NC <= a.Wc;
        const int nc = min(NC, a.Wc - cx0);
        for (int d = 0; d < dl.nd; ++d) {
            const int cd = dl.get(a, d);
            const int64_t run = cd >> 5, slot = cd & 31;
            OUT *o = reinterpret_cast<OUT *>(a.dst + run * a.run_stride + slot * a.slot_bytes) +
                     static_cast<int64_t>(y0) * a.Wp + x0;
#pragma unroll
            for (int r = 0; r < ROWS; ++r) {
                if (vl) ly[r].store(o + static_cast<int64_t>(r) * a.Wp);
                else ly[r].store_n(o + static_cast<int64_t>(r) * a.Wp, nl);
            }
            char *cb = a.dst2 + run * a.run_stride2 + slot * a.slot_bytes2;
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                OUT *q = reinterpret_cast<OUT *>(cb + p * a.cplane_bytes) + static_cast<int64_t>(cy) * a.Wc + cx0;
                if (vc) lc[p].store(q);
                else lc[p].store_n(q, nc);
            }
        }
    }
}

// NC tensor values of a row (vector when `fast`, else the first n, zeros after)
__device__ __forceinline__ void tload4(const __half *p, float (&x)[4])
{
    const uint2 v = ld_stream_v2(p);
    const float2 a = __half22float2(*reinterpret_cast<const __half2 *>(&v.x));
    const float2 b = __half22float2(*reinterpret_cast<const __half2 *>(&v.y));
    x[0] = a.x; x[1] = a.y; x[2] = b.x; x[3] = b.y;
}
__device__ __forceinline__ void tload4(const float *p, float (&x)[4])
{
    const uint4 v = ld_stream_v4(p);
    x[0] = __uint_as_float(v.x); x[1] = __uint_as_float(v.y); x[2] = __uint_as_float(v.z); x[3] = __uint_as_float(v.w);
}
template <typename TIN, int NC>
__device__ __forceinline__ void load_vals(const TIN *p, bool fast, int n, float (&x)[NC])
{
    if (fast) {
        if constexpr (NC == 8) tload8_stream(p, x);
        else tload4(p, x);
    } else {
#pragma unroll
        for (int k = 0; k < NC; ++k) x[k] = k < n ? tload1(p + k) : 0.f;
    }
}

template <typename OS, int NC>
__device__ __forceinline__ void store_codes(OS *p, const uint32_t (&q)[NC], bool vec, int n)
{
    if (vec) {
        if constexpr (NC == 8) store_samples8(p, q);
        else store_samples4(p, q);
    } else {
        store_samples_n(p, q, n);
    }
}

template <int FAMILY, typename OS, typename TIN, typename AR>
__global__ void __launch_bounds__(kThreads) t2f_yuv_generic(const T2FArgs a)
{
    constexpr bool SUB = FAMILY == kYUV420;
    constexpr int ROWS = SUB ? 2 : 1, NC = SUB ? 4 : 8;
    const T2FConst<AR> c(a.col);
    const int64_t lplane = a.th * a.tw, cplane = a.thc * a.twc;
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
        const int nvalid = min(kPx, a.Wo - x0);
        const bool full = nvalid == kPx;
        // luma: code = rne(clamp(Y' * ys + yo))  (quant_direct: exact fp16 ties)
        const TIN *ls = reinterpret_cast<const TIN *>(a.src + static_cast<int64_t>(tup) * a.tensor_stride) +
                        static_cast<int64_t>(o) * lplane + static_cast<int64_t>(y0) * a.tw + x0;
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            float v[kPx];
            load_vals<TIN, kPx>(ls + static_cast<int64_t>(r) * a.tw, a.vec_in && full, nvalid, v);
            uint32_t q[kPx];
#pragma unroll
            for (int k = 0; k < kPx; ++k) q[k] = quant_direct(static_cast<AR>(v[k]), c.yd, c.yod, c.maxc);
            store_codes<OS, kPx>(row_ptr_w<OS>(f, 0, y0 + r) + x0, q, a.vec_out && full, nvalid);
        }
        // chroma: code = rne(clamp(U * cs + (co - cs/2)))
        const int cy = SUB ? ru : y0, cx0 = SUB ? x0 >> 1 : x0, ncv = SUB ? nvalid >> 1 : nvalid;
        const TIN *cs_ = reinterpret_cast<const TIN *>(a.src2 + static_cast<int64_t>(tup) * a.tensor_stride2) +
                         static_cast<int64_t>(2 * o) * cplane + static_cast<int64_t>(cy) * a.twc + cx0;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            float v[NC];
            load_vals<TIN, NC>(cs_ + p * cplane, a.vec_in_c && full, ncv, v);
            uint32_t q[NC];
#pragma unroll
            for (int k = 0; k < NC; ++k) q[k] = quant_direct(static_cast<AR>(v[k]), c.csd, c.co2d, c.maxc);
            store_codes<OS, NC>(row_ptr_w<OS>(f, 1 + p, cy) + cx0, q, a.vec_out && full, ncv);
        }
    }
}

int sms()
{
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    }
    return n;
}

template <typename K, typename A>
cudaError_t launch(K kernel, const A &a, cudaStream_t s)
{
    if (a.items <= 0) return cudaSuccess;
    const int64_t tiles = (a.items + kThreads - 1) / kThreads;
    const int grid = static_cast<int>(std::min<int64_t>(tiles, static_cast<int64_t>(sms()) * 16));
    kernel<<<grid, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

template <int FAMILY>
cudaError_t f2t_family(int bits, int dtype, const F2TArgs &a, cudaStream_t s)
{
    if (bits == 8) {
        if (dtype == kF16) return launch(f2t_yuv_generic<FAMILY, uint8_t, __half>, a, s);
        return launch(f2t_yuv_generic<FAMILY, uint8_t, float>, a, s);
    }
    if (dtype == kF16) return launch(f2t_yuv_generic<FAMILY, uint16_t, __half>, a, s);
    return launch(f2t_yuv_generic<FAMILY, uint16_t, float>, a, s);
}

template <int FAMILY>
cudaError_t t2f_family(int bits, int dtype, const T2FArgs &a, cudaStream_t s)
{
    if (bits == 8) {
        if (dtype == kF16) return launch(t2f_yuv_generic<FAMILY, uint8_t, __half, float>, a, s);
        return launch(t2f_yuv_generic<FAMILY, uint8_t, float, float>, a, s);
    }
    if (bits == 10) {
        if (dtype == kF16) return launch(t2f_yuv_generic<FAMILY, uint16_t, __half, float>, a, s);
        return launch(t2f_yuv_generic<FAMILY, uint16_t, float, float>, a, s);
    }
    // 16-bit codes in fp64, as for RGB tensors (SURVEY.md §7 "Numerics at 16-bit")
    if (dtype == kF16) return launch(t2f_yuv_generic<FAMILY, uint16_t, __half, double>, a, s);
    return launch(t2f_yuv_generic<FAMILY, uint16_t, float, double>, a, s);
}

}  // namespace

cudaError_t launch_f2t_yuv(int family, int bits, int dtype, const F2TArgs &a, cudaStream_t s)
{
    if (a.tma_ok && (family == kYUV420 || family == kYUV444)) return launch_f2t_yuv_tma(family, bits, dtype, a, s);
    if (family == kYUV420) return f2t_family<kYUV420>(bits, dtype, a, s);
    if (family == kYUV444) return f2t_family<kYUV444>(bits, dtype, a, s);
    return cudaErrorInvalidValue;
}

cudaError_t launch_t2f_yuv(int family, int bits, int dtype, const T2FArgs &a, cudaStream_t s)
{
    if (a.tma_ok && (family == kYUV420 || family == kYUV444)) return launch_t2f_yuv_tma(family, bits, dtype, a, s);
    if (family == kYUV420) return t2f_family<kYUV420>(bits, dtype, a, s);
    if (family == kYUV444) return t2f_family<kYUV444>(bits, dtype, a, s);
    return cudaErrorInvalidValue;
}

}  // namespace nnvisr
