// kernels.cu -- sm_100a conversion kernels of the NNVISR frame<->tensor path.
//
// f2t: frames -> NCHW tensor (steps A3-A7 of SURVEY.md §8(a); §3.1
//      P:282-304 pixel format / colourspace, §3.3 P:377-379 per-slot layout).
// t2f: NCHW tensor -> frames (steps B1-B4; north_star "RGB->YUV matrix,
//      chroma downsampling, scale, round-half-even and clamp").
//
// Both are streaming HBM-bound passes (~1-3 flop/byte, no dense contraction,
// so no tensor cores).  One thread owns ROWS luma rows x 8 columns:
//   * 128-bit non-allocating loads of the packed integer planes / tensor rows;
//   * 4:2:0 chroma: the thread's 4 co-sited chroma samples per row arrive in
//     one 8/4-byte load, the two halo samples come from the neighbouring
//     threads' loads through L1; the upsample is exact integer arithmetic
//     (9a+3b+3c+d, reading A5) so fp32 sees one rounding per value;
//   * t2f: the 2x2 chroma block of a row pair lives in one thread, so the box
//     filter is an in-register add (no shuffles, no shared memory);
//   * 128-bit stores of fp16 x8 / fp32 x4 tensor rows and of output samples.
// Threads at the right edge (padding columns, widths not a multiple of 8) and
// frames whose planes are not 16-byte aligned take a scalar path that clamps
// every coordinate; the arithmetic is identical.
#include <cuda_fp16.h>

#include "internal.h"

namespace nnvisr {
namespace {

// ------------------------------------------------------------------ memory
__device__ __forceinline__ uint4 ld_stream_v4(const void *p)
{
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ uint2 ld_stream_v2(const void *p)
{
    uint2 r;
    asm("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ uint2 ld_v2(const void *p)
{
    uint2 r;
    asm("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t ld_v1(const void *p)
{
    uint32_t r;
    asm("ld.global.nc.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

template <typename T>
__device__ __forceinline__ const T *row_ptr(const DevFrame &f, int p, int y)
{
    return reinterpret_cast<const T *>(static_cast<const char *>(f.plane[p]) +
                                       static_cast<int64_t>(y) * f.pitch[p]);
}
template <typename T>
__device__ __forceinline__ T *row_ptr_w(const DevFrame &f, int p, int y)
{
    return reinterpret_cast<T *>(const_cast<char *>(static_cast<const char *>(f.plane[p])) +
                                 static_cast<int64_t>(y) * f.pitch[p]);
}

// 8 consecutive samples (16-byte aligned for u16, 8-byte for u8), streamed.
__device__ __forceinline__ void load8(const uint16_t *p, int (&v)[kPx])
{
    uint4 q = ld_stream_v4(p);
    v[0] = q.x & 0xffff; v[1] = q.x >> 16; v[2] = q.y & 0xffff; v[3] = q.y >> 16;
    v[4] = q.z & 0xffff; v[5] = q.z >> 16; v[6] = q.w & 0xffff; v[7] = q.w >> 16;
}
__device__ __forceinline__ void load8(const uint8_t *p, int (&v)[kPx])
{
    uint2 q = ld_stream_v2(p);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[k] = (q.x >> (8 * k)) & 0xff;
        v[k + 4] = (q.y >> (8 * k)) & 0xff;
    }
}
// 4 consecutive chroma samples, L1-cached (neighbours read the halo).
__device__ __forceinline__ void load4(const uint16_t *p, int *v)
{
    uint2 q = ld_v2(p);
    v[0] = q.x & 0xffff; v[1] = q.x >> 16; v[2] = q.y & 0xffff; v[3] = q.y >> 16;
}
__device__ __forceinline__ void load4(const uint8_t *p, int *v)
{
    uint32_t q = ld_v1(p);
    v[0] = q & 0xff; v[1] = (q >> 8) & 0xff; v[2] = (q >> 16) & 0xff; v[3] = q >> 24;
}
__device__ __forceinline__ int load1(const uint16_t *p) { return __ldg(p); }
__device__ __forceinline__ int load1(const uint8_t *p) { return __ldg(p); }

// ------------------------------------------------------------ tensor store
__device__ __forceinline__ uint32_t pack_half2(float a, float b)
{
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}
// ------------------------------------------------------------- tensor load
__device__ __forceinline__ void tload8(const __half *p, float (&v)[kPx])
{
    uint4 q = ld_stream_v4(p);
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&w[k]));
        v[2 * k] = f.x;
        v[2 * k + 1] = f.y;
    }
}
__device__ __forceinline__ void tload8(const float *p, float (&v)[kPx])
{
    uint4 a = ld_stream_v4(p), b = ld_stream_v4(p + 4);
    v[0] = __uint_as_float(a.x); v[1] = __uint_as_float(a.y);
    v[2] = __uint_as_float(a.z); v[3] = __uint_as_float(a.w);
    v[4] = __uint_as_float(b.x); v[5] = __uint_as_float(b.y);
    v[6] = __uint_as_float(b.z); v[7] = __uint_as_float(b.w);
}
__device__ __forceinline__ float tload1(const __half *p) { return __half2float(p[0]); }
__device__ __forceinline__ float tload1(const float *p) { return __ldg(p); }

// ------------------------------------------------------------ f2t colour
// Steps A5-A6: dequantise (exact integer offset, one fp32 rounding) and the
// inverse matrix with no clamp (reading A4).
template <int FAMILY>
__device__ __forceinline__ void f2t_colour(const F2TColour &c, int ys, int us, int vs, float &R,
                                           float &G, float &B)
{
    if (FAMILY == kRGB) {
        R = static_cast<float>(ys - c.y_off) * c.y_scale;
        G = static_cast<float>(us - c.y_off) * c.y_scale;
        B = static_cast<float>(vs - c.y_off) * c.y_scale;
    } else {
        const float Y = static_cast<float>(ys - c.y_off) * c.y_scale;
        const float Pb = static_cast<float>(us - c.c_off) * c.c_scale;
        const float Pr = static_cast<float>(vs - c.c_off) * c.c_scale;
        R = fmaf(c.r_pr, Pr, Y);
        B = fmaf(c.b_pb, Pb, Y);
        G = fmaf(-c.g_pr, Pr, fmaf(-c.g_pb, Pb, Y));
    }
}

// fp16 tensors near zero: a difference of O(1) terms rounded in fp32 can be
// off by more than one fp16 ULP once |v| < 2^-9 (the ULP there is < 2^-19).
// Those (rare) pixels are recomputed in fp64 and rounded once to fp16; the
// returned float is that fp16 value exactly, so the RNE store reproduces it.
__device__ __forceinline__ float3 f2t_colour_precise(const F2TColour &c, int ys, int us, int vs)
{
    const double Y = static_cast<double>(ys - c.y_off) * c.y_scale_d;
    const double Pb = static_cast<double>(us - c.c_off) * c.c_scale_d;
    const double Pr = static_cast<double>(vs - c.c_off) * c.c_scale_d;
    return make_float3(__half2float(__double2half(Y + c.r_pr_d * Pr)),
                       __half2float(__double2half(Y - c.g_pb_d * Pb - c.g_pr_d * Pr)),
                       __half2float(__double2half(Y + c.b_pb_d * Pb)));
}

template <int FAMILY, typename OUT>
__device__ __forceinline__ void f2t_pixel(const F2TColour &c, int ys, int us, int vs, float &R, float &G,
                                          float &B)
{
    f2t_colour<FAMILY>(c, ys, us, vs, R, G, B);
    if (FAMILY != kRGB && sizeof(OUT) == 2) {
        constexpr float kTiny = 1.0f / 512.0f;
        if (fabsf(R) < kTiny || fabsf(G) < kTiny || fabsf(B) < kTiny) {
            const float3 p = f2t_colour_precise(c, ys, us, vs);
            R = p.x;
            G = p.y;
            B = p.z;
        }
    }
}

// Scalar path: sample codes of pixel (x, y) with every coordinate clamped
// (padding replicates the last row/column, reading A6; chroma taps clamp to
// the plane, reading A5).  Values are 16 x code.
template <int FAMILY, typename IN>
__device__ __forceinline__ void f2t_codes_scalar(const DevFrame &f, int W, int H, int x, int y,
                                                 int &ys, int &us, int &vs)
{
    const int xc = min(x, W - 1), yc = min(y, H - 1);
    ys = 16 * load1(row_ptr<IN>(f, 0, yc) + xc);
    if (FAMILY == kYUV420) {
        const int cw = W >> 1, ch = H >> 1;
        const int jn = yc >> 1, jf = (yc & 1) ? min(jn + 1, ch - 1) : max(jn - 1, 0);
        const int in_ = xc >> 1, if_ = (xc & 1) ? min(in_ + 1, cw - 1) : max(in_ - 1, 0);
        const IN *u0 = row_ptr<IN>(f, 1, jn), *u1 = row_ptr<IN>(f, 1, jf);
        const IN *v0 = row_ptr<IN>(f, 2, jn), *v1 = row_ptr<IN>(f, 2, jf);
        us = 9 * load1(u0 + in_) + 3 * load1(u0 + if_) + 3 * load1(u1 + in_) + load1(u1 + if_);
        vs = 9 * load1(v0 + in_) + 3 * load1(v0 + if_) + 3 * load1(v1 + in_) + load1(v1 + if_);
    } else {
        us = 16 * load1(row_ptr<IN>(f, 1, yc) + xc);
        vs = 16 * load1(row_ptr<IN>(f, 2, yc) + xc);
    }
}

// Horizontal 2x upsample of one chroma row around the thread's 8 columns:
// c[0] = sample i0-1 (clamped), c[1..4] = i0..i0+3, c[5] = i0+4 (clamped).
// Even luma column 2m: 3*c[m+1] + c[m];  odd 2m+1: 3*c[m+1] + c[m+2].
__device__ __forceinline__ void hup(const int (&c)[6], int (&h)[kPx])
{
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        h[2 * m] = 3 * c[m + 1] + c[m];
        h[2 * m + 1] = 3 * c[m + 1] + c[m + 2];
    }
}

template <typename IN>
__device__ __forceinline__ void chroma_row6(const IN *row, int i0, int cw, int (&c)[6])
{
    load4(row + i0, &c[1]);
    c[0] = load1(row + max(i0 - 1, 0));
    c[5] = load1(row + min(i0 + 4, cw - 1));
}

// Packed tensor values of one row of 8 pixels and one channel.
template <typename OUT> struct Row8;
template <> struct Row8<__half> {
    uint4 v;
    __device__ __forceinline__ void set(const float (&x)[kPx])
    {
        v = make_uint4(pack_half2(x[0], x[1]), pack_half2(x[2], x[3]), pack_half2(x[4], x[5]),
                       pack_half2(x[6], x[7]));
    }
    __device__ __forceinline__ void store(__half *p) const { *reinterpret_cast<uint4 *>(p) = v; }
    __device__ __forceinline__ void store_n(__half *p, int n) const
    {
        const __half *h = reinterpret_cast<const __half *>(&v);
        for (int k = 0; k < n; ++k) p[k] = h[k];
    }
};
template <> struct Row8<float> {
    float4 a, b;
    __device__ __forceinline__ void set(const float (&x)[kPx])
    {
        a = make_float4(x[0], x[1], x[2], x[3]);
        b = make_float4(x[4], x[5], x[6], x[7]);
    }
    __device__ __forceinline__ void store(float *p) const
    {
        reinterpret_cast<float4 *>(p)[0] = a;
        reinterpret_cast<float4 *>(p)[1] = b;
    }
    __device__ __forceinline__ void store_n(float *p, int n) const
    {
        const float x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        for (int k = 0; k < n; ++k) p[k] = x[k];
    }
};

// One thread: ROWS rows x 8 columns of one distinct frame, converted once and
// stored to every (run, slot) of the launch that holds this frame (a frame
// shared by N overlapping windows, or repeated inside a tuple at a scene cut,
// is read and converted once: PAPER.md §3.3 P:373-377's point that a batch
// only has b*n+1 distinct frames).
template <int FAMILY, typename IN, typename OUT>
__global__ void __launch_bounds__(kThreads) f2t_kernel(const F2TArgs a)
{
    constexpr int ROWS = (FAMILY == kYUV420) ? 2 : 1;
    const int unit = blockIdx.x * kThreads + threadIdx.x;
    if (unit >= a.units) return;
    const int job = a.job_base + blockIdx.y;
    const int ru = unit / a.col_units;
    const int x0 = (unit - ru * a.col_units) * kPx;
    const int y0 = ru * ROWS;
    const DevFrame f = a.frames[a.job_frame[job]];

    int ys[ROWS][kPx], us[ROWS][kPx], vs[ROWS][kPx];
    int yc[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) yc[r] = min(y0 + r, a.H - 1);

    if (a.vec_in && x0 + kPx <= a.W) {
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            load8(row_ptr<IN>(f, 0, yc[r]) + x0, ys[r]);
#pragma unroll
            for (int k = 0; k < kPx; ++k) ys[r][k] *= 16;
        }
        if (FAMILY == kYUV420) {
            const int cw = a.W >> 1, ch = a.H >> 1, i0 = x0 >> 1;
            // the near chroma row is shared by both luma rows; far rows differ
            const int jn = yc[0] >> 1;
            int jf[ROWS];
#pragma unroll
            for (int r = 0; r < ROWS; ++r)
                jf[r] = (yc[r] & 1) ? min((yc[r] >> 1) + 1, ch - 1) : max((yc[r] >> 1) - 1, 0);
#pragma unroll
            for (int p = 1; p <= 2; ++p) {
                int cn[6], hn[kPx];
                chroma_row6(row_ptr<IN>(f, p, jn), i0, cw, cn);
                hup(cn, hn);
#pragma unroll
                for (int r = 0; r < ROWS; ++r) {
                    int cf[6], hf[kPx];
                    chroma_row6(row_ptr<IN>(f, p, jf[r]), i0, cw, cf);
                    hup(cf, hf);
#pragma unroll
                    for (int k = 0; k < kPx; ++k) {
                        const int sm = 3 * hn[k] + hf[k];
                        if (p == 1) us[r][k] = sm; else vs[r][k] = sm;
                    }
                }
            }
        } else {
#pragma unroll
            for (int r = 0; r < ROWS; ++r) {
                load8(row_ptr<IN>(f, 1, yc[r]) + x0, us[r]);
                load8(row_ptr<IN>(f, 2, yc[r]) + x0, vs[r]);
#pragma unroll
                for (int k = 0; k < kPx; ++k) { us[r][k] *= 16; vs[r][k] *= 16; }
            }
        }
    } else {
#pragma unroll
        for (int r = 0; r < ROWS; ++r)
#pragma unroll
            for (int k = 0; k < kPx; ++k)
                f2t_codes_scalar<FAMILY, IN>(f, a.W, a.H, x0 + k, y0 + r, ys[r][k], us[r][k], vs[r][k]);
    }

    Row8<OUT> out[ROWS][3];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        float R[kPx], G[kPx], B[kPx];
#pragma unroll
        for (int k = 0; k < kPx; ++k) f2t_pixel<FAMILY, OUT>(a.col, ys[r][k], us[r][k], vs[r][k], R[k], G[k], B[k]);
        out[r][0].set(R);
        out[r][1].set(G);
        out[r][2].set(B);
    }

    const int64_t plane = static_cast<int64_t>(a.Hp) * a.Wp;
    const int64_t off = static_cast<int64_t>(y0) * a.Wp + x0;
    const bool vec_store = a.vec_out && (x0 + kPx <= a.Wp);
    const int d1 = a.job_dst[job + 1];
    for (int d = a.job_dst[job]; d < d1; ++d) {
        const int code = a.dst_code[d];
        OUT *o = reinterpret_cast<OUT *>(a.dst + static_cast<int64_t>(code >> 5) * a.run_stride +
                                         static_cast<int64_t>(code & 31) * a.slot_bytes) + off;
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                OUT *q = o + c * plane + static_cast<int64_t>(r) * a.Wp;
                if (vec_store) out[r][c].store(q);
                else out[r][c].store_n(q, min(kPx, a.Wp - x0));
            }
        }
    }
}

// ------------------------------------------------------------ t2f colour
template <typename T> struct T2FConst;
template <> struct T2FConst<float> {
    float kr, kb, db, dr, idb, idr, ys, yo, cs, co, maxc;
    __device__ explicit T2FConst(const T2FColour &c)
        : kr(c.fkr), kb(c.fkb), db(c.fdb), dr(c.fdr), idb(c.fidb), idr(c.fidr), ys(c.fys), yo(c.fyo),
          cs(c.fcs), co(c.fco), maxc(c.fmaxc) {}
};
template <> struct T2FConst<double> {
    double kr, kb, db, dr, idb, idr, ys, yo, cs, co, maxc;
    __device__ explicit T2FConst(const T2FColour &c)
        : kr(c.kr), kb(c.kb), db(c.db), dr(c.dr), idb(c.idb), idr(c.idr), ys(c.ys), yo(c.yo), cs(c.cs),
          co(c.co), maxc(c.maxc) {}
};

__device__ __forceinline__ float fma_(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fma_(double a, double b, double c) { return fma(a, b, c); }

// Step B4: clamp to [0, maxc] (NaN -> 0: fmax returns the non-NaN operand),
// then round half to even by adding 1.5 * 2^(p-1): the sum lies where the
// spacing of representable values is exactly 1, so the FP add rounds the
// value to the nearest integer, ties to even, and the integer is the low bits.
__device__ __forceinline__ uint32_t quant(float q, float maxc)
{
    const float x = fminf(fmaxf(q, 0.0f), maxc);
    return __float_as_uint(x + 12582912.0f) - 0x4B400000u;
}
__device__ __forceinline__ uint32_t quant(double q, double maxc)
{
    const double x = fmin(fmax(q, 0.0), maxc);
    return static_cast<uint32_t>(__double2loint(x + 6755399441055744.0));
}

// S / d for a divisor d with precomputed reciprocal id: one FMA correction of
// the reciprocal product (correctly rounded quotient; keeps exact quotients
// such as the full-range primaries' +-0.5 exact).
template <typename T>
__device__ __forceinline__ T divide(T S, T d, T id)
{
    const T q0 = S * id;
    const T r = fma_(-q0, d, S);
    return fma_(r, id, q0);
}

__device__ __forceinline__ void store_samples8(uint16_t *p, const uint32_t (&v)[kPx])
{
    *reinterpret_cast<uint4 *>(p) = make_uint4(__byte_perm(v[0], v[1], 0x5410), __byte_perm(v[2], v[3], 0x5410),
                                               __byte_perm(v[4], v[5], 0x5410), __byte_perm(v[6], v[7], 0x5410));
}
__device__ __forceinline__ uint32_t pack4_u8(uint32_t a, uint32_t b, uint32_t c, uint32_t d)
{
    return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}
__device__ __forceinline__ void store_samples8(uint8_t *p, const uint32_t (&v)[kPx])
{
    *reinterpret_cast<uint2 *>(p) = make_uint2(pack4_u8(v[0], v[1], v[2], v[3]), pack4_u8(v[4], v[5], v[6], v[7]));
}
__device__ __forceinline__ void store_samples4(uint16_t *p, const uint32_t *v)
{
    *reinterpret_cast<uint2 *>(p) = make_uint2(__byte_perm(v[0], v[1], 0x5410), __byte_perm(v[2], v[3], 0x5410));
}
__device__ __forceinline__ void store_samples4(uint8_t *p, const uint32_t *v)
{
    *reinterpret_cast<uint32_t *>(p) = pack4_u8(v[0], v[1], v[2], v[3]);
}

template <int FAMILY, typename OS, typename TIN, typename AR>
__global__ void __launch_bounds__(kThreads) t2f_kernel(const T2FArgs a)
{
    constexpr int ROWS = (FAMILY == kYUV420) ? 2 : 1;
    const int unit = blockIdx.x * kThreads + threadIdx.x;
    if (unit >= a.units) return;
    const int job = a.job_base + blockIdx.y;
    const int tup = job / a.M, o = job - tup * a.M;
    const int ru = unit / a.col_units;
    const int x0 = (unit - ru * a.col_units) * kPx;
    const int y0 = ru * ROWS;
    const int64_t plane = a.th * a.tw;
    const TIN *src = reinterpret_cast<const TIN *>(a.src + static_cast<int64_t>(tup) * a.tensor_stride) +
                     static_cast<int64_t>(3 * o) * plane;
    const DevFrame f = a.out[job];
    const int nvalid = min(kPx, a.Wo - x0);
    const bool full = nvalid == kPx;

    // Step B1: the thread's 2x8 (4:2:0) or 1x8 window of R', G', B'
    float R[ROWS][kPx], G[ROWS][kPx], B[ROWS][kPx];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        const TIN *row = src + static_cast<int64_t>(y0 + r) * a.tw + x0;
        if (a.vec_in && full) {
            tload8(row, R[r]);
            tload8(row + plane, G[r]);
            tload8(row + 2 * plane, B[r]);
        } else {
#pragma unroll
            for (int k = 0; k < kPx; ++k) {
                const bool in = k < nvalid;
                R[r][k] = in ? tload1(row + k) : 0.f;
                G[r][k] = in ? tload1(row + plane + k) : 0.f;
                B[r][k] = in ? tload1(row + 2 * plane + k) : 0.f;
            }
        }
    }

    const T2FConst<AR> c(a.col);
    const bool vec_store = a.vec_out && full;
    if (FAMILY == kRGB) {
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            uint32_t q[3][kPx];
#pragma unroll
            for (int k = 0; k < kPx; ++k) {
                q[0][k] = quant(fma_(static_cast<AR>(R[r][k]), c.ys, c.yo), c.maxc);
                q[1][k] = quant(fma_(static_cast<AR>(G[r][k]), c.ys, c.yo), c.maxc);
                q[2][k] = quant(fma_(static_cast<AR>(B[r][k]), c.ys, c.yo), c.maxc);
            }
#pragma unroll
            for (int p = 0; p < 3; ++p) {
                OS *out = row_ptr_w<OS>(f, p, y0 + r) + x0;
                if (vec_store) store_samples8(out, q[p]);
                else for (int k = 0; k < nvalid; ++k) out[k] = static_cast<OS>(q[p][k]);
            }
        }
        return;
    }

    // Step B2 (luma) + B4: Y' = G + Kr(R-G) + Kb(B-G); keep B-Y', R-Y'
    AR BY[ROWS][kPx], RY[ROWS][kPx];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        uint32_t qy[kPx];
#pragma unroll
        for (int k = 0; k < kPx; ++k) {
            const AR r_ = R[r][k], g_ = G[r][k], b_ = B[r][k];
            const AR Y = fma_(c.kb, b_ - g_, fma_(c.kr, r_ - g_, g_));
            BY[r][k] = b_ - Y;
            RY[r][k] = r_ - Y;
            qy[k] = quant(fma_(Y, c.ys, c.yo), c.maxc);
        }
        OS *out = row_ptr_w<OS>(f, 0, y0 + r) + x0;
        if (vec_store) store_samples8(out, qy);
        else for (int k = 0; k < nvalid; ++k) out[k] = static_cast<OS>(qy[k]);
    }

    if (FAMILY == kYUV444) {
        uint32_t qb[kPx], qr[kPx];
#pragma unroll
        for (int k = 0; k < kPx; ++k) {
            qb[k] = quant(fma_(divide(BY[0][k], c.db, c.idb), c.cs, c.co), c.maxc);
            qr[k] = quant(fma_(divide(RY[0][k], c.dr, c.idr), c.cs, c.co), c.maxc);
        }
        OS *ob = row_ptr_w<OS>(f, 1, y0) + x0, *orr = row_ptr_w<OS>(f, 2, y0) + x0;
        if (vec_store) { store_samples8(ob, qb); store_samples8(orr, qr); }
        else for (int k = 0; k < nvalid; ++k) { ob[k] = static_cast<OS>(qb[k]); orr[k] = static_cast<OS>(qr[k]); }
        return;
    }

    // Step B3: 2x2 box mean, ((a+b)+(c+d))/4, folded into the divisor 4*db
    // (a power-of-two scaling, exact): Pb = S / (4 db), Pr = S / (4 dr).
    const AR db4 = c.db * AR(4), dr4 = c.dr * AR(4), idb4 = c.idb * AR(0.25), idr4 = c.idr * AR(0.25);
    uint32_t qb[4], qr[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const int r1 = ROWS - 1;
        const AR sb = (BY[0][2 * m] + BY[0][2 * m + 1]) + (BY[r1][2 * m] + BY[r1][2 * m + 1]);
        const AR sr = (RY[0][2 * m] + RY[0][2 * m + 1]) + (RY[r1][2 * m] + RY[r1][2 * m + 1]);
        qb[m] = quant(fma_(divide(sb, db4, idb4), c.cs, c.co), c.maxc);
        qr[m] = quant(fma_(divide(sr, dr4, idr4), c.cs, c.co), c.maxc);
    }
    OS *ob = row_ptr_w<OS>(f, 1, y0 >> 1) + (x0 >> 1), *orr = row_ptr_w<OS>(f, 2, y0 >> 1) + (x0 >> 1);
    if (vec_store) { store_samples4(ob, qb); store_samples4(orr, qr); }
    else for (int m = 0; m < nvalid / 2; ++m) { ob[m] = static_cast<OS>(qb[m]); orr[m] = static_cast<OS>(qr[m]); }
}

dim3 grid_for(int units, int jobs) { return dim3((units + kThreads - 1) / kThreads, jobs); }

template <int FAMILY>
cudaError_t f2t_dispatch(int bits, int dtype, const F2TArgs &a, int jobs, cudaStream_t s)
{
    const dim3 g = grid_for(a.units, jobs);
    if (bits == 8) {
        if (dtype == kF16) f2t_kernel<FAMILY, uint8_t, __half><<<g, kThreads, 0, s>>>(a);
        else f2t_kernel<FAMILY, uint8_t, float><<<g, kThreads, 0, s>>>(a);
    } else {
        if (dtype == kF16) f2t_kernel<FAMILY, uint16_t, __half><<<g, kThreads, 0, s>>>(a);
        else f2t_kernel<FAMILY, uint16_t, float><<<g, kThreads, 0, s>>>(a);
    }
    return cudaGetLastError();
}

template <int FAMILY>
cudaError_t t2f_dispatch(int bits, int dtype, const T2FArgs &a, int jobs, cudaStream_t s)
{
    const dim3 g = grid_for(a.units, jobs);
    if (bits == 8) {
        if (dtype == kF16) t2f_kernel<FAMILY, uint8_t, __half, float><<<g, kThreads, 0, s>>>(a);
        else t2f_kernel<FAMILY, uint8_t, float, float><<<g, kThreads, 0, s>>>(a);
    } else if (bits == 10) {
        if (dtype == kF16) t2f_kernel<FAMILY, uint16_t, __half, float><<<g, kThreads, 0, s>>>(a);
        else t2f_kernel<FAMILY, uint16_t, float, float><<<g, kThreads, 0, s>>>(a);
    } else {
        // 16-bit codes: fp32 arithmetic leaves ~0.2% of codes 1 LSB off the
        // exact result, so B2/B4 run in fp64 (SURVEY.md §7 "Numerics at 16-bit").
        if (dtype == kF16) t2f_kernel<FAMILY, uint16_t, __half, double><<<g, kThreads, 0, s>>>(a);
        else t2f_kernel<FAMILY, uint16_t, float, double><<<g, kThreads, 0, s>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_f2t(int family, int bits, int dtype, const F2TArgs &a, int jobs, cudaStream_t s)
{
    count_launch();
    switch (family) {
    case kYUV420: return f2t_dispatch<kYUV420>(bits, dtype, a, jobs, s);
    case kYUV444: return f2t_dispatch<kYUV444>(bits, dtype, a, jobs, s);
    default: return f2t_dispatch<kRGB>(bits, dtype, a, jobs, s);
    }
}

cudaError_t launch_t2f(int family, int bits, int dtype, const T2FArgs &a, int jobs, cudaStream_t s)
{
    count_launch();
    switch (family) {
    case kYUV420: return t2f_dispatch<kYUV420>(bits, dtype, a, jobs, s);
    case kYUV444: return t2f_dispatch<kYUV444>(bits, dtype, a, jobs, s);
    default: return t2f_dispatch<kRGB>(bits, dtype, a, jobs, s);
    }
}

}  // namespace nnvisr
