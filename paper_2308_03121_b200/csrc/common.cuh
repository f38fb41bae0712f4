// common.cuh -- device helpers shared by the generic (LDG) and the TMA
// pipelined conversion kernels: memory access, the colour arithmetic of
// steps A5-A6 (frames -> tensor) and B2-B4 (tensor -> frames), packing.
#pragma once

#include <cuda_fp16.h>

#include <cstdio>

#include "internal.h"

namespace nnvisr {
namespace dev {

// ------------------------------------------------------------ checked builds
// `make checked` (-DNNVISR_CHECKED, libnnvisr_checked.so): compute-sanitizer
// is closed on the GPU pool, so the kernels check their own accesses -- every
// shared-memory vector access of the staging kernels lies inside the dynamic
// shared memory, every TMA copy is 16-byte aligned and, in f2t, lands inside
// its stage / reads inside its output buffer and a bound frame's planes.  A
// failed check prints the site and traps (the launch fails loudly).
#ifdef NNVISR_CHECKED
extern __shared__ __align__(16) uint8_t nnvisr_dsmem[];  // aliases every kernel's dynamic smem
__device__ __forceinline__ bool smem_ok(const void *p, uint32_t n)
{
    if (!__isShared(p)) return true;
    uint32_t dyn;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    const uint32_t o = static_cast<uint32_t>(__cvta_generic_to_shared(p));
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(nnvisr_dsmem));
    return o >= b && o + n <= b + dyn;
}
#define NNVISR_CHECK(cond)                                                                                   \
    do {                                                                                                     \
        if (!(cond)) {                                                                                       \
            printf("nnvisr check failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond,       \
                   (int)blockIdx.x, (int)threadIdx.x);                                                       \
            __trap();                                                                                        \
        }                                                                                                    \
    } while (0)
#define NNVISR_CHECK_SMEM(p, n) NNVISR_CHECK(::nnvisr::dev::smem_ok((p), (n)))
#else
#define NNVISR_CHECK(cond) \
    do {                   \
    } while (0)
#define NNVISR_CHECK_SMEM(p, n) NNVISR_CHECK(true)
#endif

// ------------------------------------------------------------------ memory
__device__ __forceinline__ uint4 ld_stream_v4(const void *p)
{
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ uint2 ld_stream_v2(const void *p)
{
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ uint2 ld_v2(const void *p)
{
    uint2 r;
    asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t ld_v1(const void *p)
{
    uint32_t r;
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ int load1(const uint16_t *p) { return __ldg(p); }
__device__ __forceinline__ int load1(const uint8_t *p) { return __ldg(p); }

__device__ __forceinline__ DevFrame load_frame(const DevFrame *p)
{
    DevFrame f;
    const uint4 a = __ldg(reinterpret_cast<const uint4 *>(p));
    const uint4 b = __ldg(reinterpret_cast<const uint4 *>(p) + 1);
    const uint4 c = __ldg(reinterpret_cast<const uint4 *>(p) + 2);
    f.plane[0] = reinterpret_cast<const void *>((uint64_t)a.x | ((uint64_t)a.y << 32));
    f.plane[1] = reinterpret_cast<const void *>((uint64_t)a.z | ((uint64_t)a.w << 32));
    f.plane[2] = reinterpret_cast<const void *>((uint64_t)b.x | ((uint64_t)b.y << 32));
    f.pitch[0] = (int64_t)((uint64_t)b.z | ((uint64_t)b.w << 32));
    f.pitch[1] = (int64_t)((uint64_t)c.x | ((uint64_t)c.y << 32));
    f.pitch[2] = (int64_t)((uint64_t)c.z | ((uint64_t)c.w << 32));
    return f;
}

template <typename T>
__device__ __forceinline__ const T *row_ptr(const DevFrame &f, int p, int y)
{
    return reinterpret_cast<const T *>(static_cast<const char *>(f.plane[p]) + static_cast<int64_t>(y) * f.pitch[p]);
}
template <typename T>
__device__ __forceinline__ T *row_ptr_w(const DevFrame &f, int p, int y)
{
    return reinterpret_cast<T *>(const_cast<char *>(static_cast<const char *>(f.plane[p])) +
                                 static_cast<int64_t>(y) * f.pitch[p]);
}

// unpack 8 / 4 packed samples
__device__ __forceinline__ void unpack8(uint4 q, int (&v)[kPx])
{
    v[0] = q.x & 0xffff; v[1] = q.x >> 16; v[2] = q.y & 0xffff; v[3] = q.y >> 16;
    v[4] = q.z & 0xffff; v[5] = q.z >> 16; v[6] = q.w & 0xffff; v[7] = q.w >> 16;
}
__device__ __forceinline__ void unpack8(uint2 q, int (&v)[kPx])
{
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[k] = (q.x >> (8 * k)) & 0xff;
        v[k + 4] = (q.y >> (8 * k)) & 0xff;
    }
}
__device__ __forceinline__ void unpack4(uint2 q, int *v)
{
    v[0] = q.x & 0xffff; v[1] = q.x >> 16; v[2] = q.y & 0xffff; v[3] = q.y >> 16;
}
__device__ __forceinline__ void unpack4(uint32_t q, int *v)
{
    v[0] = q & 0xff; v[1] = (q >> 8) & 0xff; v[2] = (q >> 16) & 0xff; v[3] = q >> 24;
}
// 8 samples / 4 samples packed in one vector of the sample type
template <typename IN> struct Pack;
template <> struct Pack<uint16_t> { using V8 = uint4; using V4 = uint2; };
template <> struct Pack<uint8_t> { using V8 = uint2; using V4 = uint32_t; };

__device__ __forceinline__ uint32_t pack_half2(float a, float b)
{
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}

// ------------------------------------------------------------ f2t colour
// Steps A5-A6: dequantise and apply the inverse matrix with no clamp (reading
// A4).  Inputs are 16 x code.  Y' = (ys - y_off) * y_scale (exact integer
// offset, one fp32 rounding); the chroma offsets are exact integers too and
// the chroma scale is folded into the matrix constants (r_v = r_pr * c_scale
// etc., each rounded once from double), so R' = Y' + r_v * (vs - c_off) is one
// FMA.
template <int FAMILY>
__device__ __forceinline__ void f2t_colour(const F2TColour &c, int ys, int us, int vs, float &R, float &G, float &B)
{
    if (FAMILY == kRGB) {
        R = static_cast<float>(ys - c.y_off) * c.y_scale;
        G = static_cast<float>(us - c.y_off) * c.y_scale;
        B = static_cast<float>(vs - c.y_off) * c.y_scale;
    } else {
        const float Y = static_cast<float>(ys - c.y_off) * c.y_scale;
        const float du = static_cast<float>(us - c.c_off), dv = static_cast<float>(vs - c.c_off);
        R = fmaf(c.r_v, dv, Y);
        B = fmaf(c.b_u, du, Y);
        G = fmaf(-c.g_v, dv, fmaf(-c.g_u, du, Y));
    }
}

// fp16 tensors near zero: R', G', B' are sums of O(1) terms whose fp32
// evaluation errs by at most ~2^-23 (one rounding of Y' <= 1.2, the rounded
// folded constants, the FMA roundings).  Against the oracle's single
// double->fp16 rounding that stays within 1 fp16 ULP while the ULP exceeds
// the error: for |v| >= 2^-11 the ULP is >= 2^-21, four times the bound.
// Pixels with a value below 2^-11 are recomputed in fp64 and rounded once to
// fp16; the returned float is that fp16 value exactly, so the RNE store
// reproduces it.  (tests/test_gpu_fp16_exhaustive.py: every 8-bit triple,
// all matrices and ranges.)
__device__ __forceinline__ float3 f2t_colour_precise(const F2TColour &c, int ys, int us, int vs)
{
    const double Y = static_cast<double>(ys - c.y_off) * c.y_scale_d;
    const double Pb = static_cast<double>(us - c.c_off) * c.c_scale_d;
    const double Pr = static_cast<double>(vs - c.c_off) * c.c_scale_d;
    return make_float3(__half2float(__double2half(Y + c.r_pr_d * Pr)),
                       __half2float(__double2half(Y - c.g_pb_d * Pb - c.g_pr_d * Pr)),
                       __half2float(__double2half(Y + c.b_pb_d * Pb)));
}
constexpr float kF16Tiny = 1.0f / 2048.0f;  // 2^-11

template <int FAMILY, typename OUT>
__device__ __forceinline__ void f2t_pixel(const F2TColour &c, int ys, int us, int vs, float &R, float &G, float &B)
{
    f2t_colour<FAMILY>(c, ys, us, vs, R, G, B);
    if (FAMILY != kRGB && sizeof(OUT) == 2) {
        if (fabsf(R) < kF16Tiny || fabsf(G) < kF16Tiny || fabsf(B) < kF16Tiny) {
            const float3 p = f2t_colour_precise(c, ys, us, vs);
            R = p.x;
            G = p.y;
            B = p.z;
        }
    }
}

// ---- float-input variant (TMA 4:2:0 fast path).  Integer samples are
// turned into floats with the magic-number trick: for 0 <= v < 2^23 the
// float with bits 0x4B000000 | v is exactly 2^23 + v, and subtracting
// (2^23 + offset) leaves the exact integer v - offset (one PRMT/LOP3 + one
// FADD instead of an I2F).  Every later step works on exact small integers
// until the colour FMAs, so the results equal the integer path bit for bit.
constexpr uint32_t kMagicBits = 0x4B000000u;
constexpr float kMagic = 8388608.0f;  // 2^23
__device__ __forceinline__ float mag(uint32_t bits) { return __uint_as_float(bits); }
// 4 packed samples -> 4 magic floats
__device__ __forceinline__ void mag4(uint2 q, float *f)  // 16-bit
{
    f[0] = mag(__byte_perm(q.x, kMagicBits, 0x7610));
    f[1] = mag(__byte_perm(q.x, kMagicBits, 0x7632));
    f[2] = mag(__byte_perm(q.y, kMagicBits, 0x7610));
    f[3] = mag(__byte_perm(q.y, kMagicBits, 0x7632));
}
__device__ __forceinline__ void mag4(uint32_t q, float *f)  // 8-bit
{
    f[0] = mag(__byte_perm(q, kMagicBits, 0x7650));
    f[1] = mag(__byte_perm(q, kMagicBits, 0x7651));
    f[2] = mag(__byte_perm(q, kMagicBits, 0x7652));
    f[3] = mag(__byte_perm(q, kMagicBits, 0x7653));
}
__device__ __forceinline__ void mag8(uint4 q, float (&f)[kPx])  // 16-bit
{
    mag4(make_uint2(q.x, q.y), f);
    mag4(make_uint2(q.z, q.w), f + 4);
}
__device__ __forceinline__ void mag8(uint2 q, float (&f)[kPx])  // 8-bit
{
    mag4(q.x, f);
    mag4(q.y, f + 4);
}

// R', G', B' from dyv = code_Y - y_off/16, du = (16x upsampled Cb) - c_off,
// dv likewise (all exact integers held in floats): the same arithmetic as
// f2t_colour (Y' = 16*dyv*y_scale exactly), fp16 near-zero values in fp64.
// fp16 near-zero values (see f2t_colour_precise): recompute the pixel in
// fp64 from dyv = code_Y - y_off/16, du = 16x Cb - c_off, dv likewise.
template <typename OUT>
__device__ __forceinline__ void f2t_fix_tiny(const F2TColour &c, float dyv, float du, float dv, float &R, float &G,
                                             float &B)
{
    if (sizeof(OUT) == 2) {
        if (fabsf(R) < kF16Tiny || fabsf(G) < kF16Tiny || fabsf(B) < kF16Tiny) {
            const double Yd = 16.0 * static_cast<double>(dyv) * c.y_scale_d;
            const double Pb = static_cast<double>(du) * c.c_scale_d, Pr = static_cast<double>(dv) * c.c_scale_d;
            R = __half2float(__double2half(Yd + c.r_pr_d * Pr));
            G = __half2float(__double2half(Yd - c.g_pb_d * Pb - c.g_pr_d * Pr));
            B = __half2float(__double2half(Yd + c.b_pb_d * Pb));
        }
    }
}

// Horizontal 2x upsample of one chroma row around an item's 8 columns:
// c[0] = sample i0-1 (clamped), c[1..4] = i0..i0+3, c[5] = i0+4 (clamped).
// Even luma column 2m: 3*c[m+1] + c[m];  odd 2m+1: 3*c[m+1] + c[m+2]
// (centre siting, reading A5; the vertical pass adds 3*near + far).
__device__ __forceinline__ void hup(const int (&c)[6], int (&h)[kPx])
{
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        h[2 * m] = 3 * c[m + 1] + c[m];
        h[2 * m + 1] = 3 * c[m + 1] + c[m + 2];
    }
}

// hup of the staged chroma row C around an item's 8 columns (i0 = x / 2):
// samples i0-1 .. i0+4, the outer two clamped to [0, cw).
template <typename IN, typename V4>
__device__ __forceinline__ void hup_row(const IN *C, int i0, int cw, int (&h)[kPx])
{
    int c[6];
    unpack4(*reinterpret_cast<const V4 *>(C + i0), &c[1]);
    c[0] = C[max(i0 - 1, 0)];
    c[5] = C[min(i0 + 4, cw - 1)];
    hup(c, h);
}

// LEFT (MPEG-2) siting: chroma i is co-sited with luma column 2i, so even
// column 2m takes 4*c[m+1] and odd 2m+1 takes 2*(c[m+1] + c[m+2]) (weights
// 1 and 1/2,1/2 scaled to the same sum 4 as hup; reading A5).
__device__ __forceinline__ void hup_left(const int (&c)[6], int (&h)[kPx])
{
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        h[2 * m] = 4 * c[m + 1];
        h[2 * m + 1] = 2 * (c[m + 1] + c[m + 2]);
    }
}

// Chroma rows of a 4:2:0 luma row y (already clamped to the frame): the near
// row and the far row (above for even y, below for odd y), clamped.
__device__ __forceinline__ int chroma_near(int yc) { return yc >> 1; }
__device__ __forceinline__ int chroma_far(int yc, int ch)
{
    return (yc & 1) ? min((yc >> 1) + 1, ch - 1) : max((yc >> 1) - 1, 0);
}

// Scalar path: sample codes of pixel (x, y) with every coordinate clamped
// (padding replicates the last row/column, reading A6; chroma taps clamp to
// the plane, reading A5).  Values are 16 x code.
template <int FAMILY, typename IN>
__device__ __forceinline__ void f2t_codes_scalar(const DevFrame &f, int W, int H, int x, int y, int &ys, int &us,
                                                 int &vs, int left = 0)
{
    const int xc = min(x, W - 1), yc = min(y, H - 1);
    ys = 16 * load1(row_ptr<IN>(f, 0, yc) + xc);
    if (FAMILY == kYUV420) {
        const int cw = W >> 1, ch = H >> 1;
        const int jn = chroma_near(yc), jf = chroma_far(yc, ch);
        const int in_ = xc >> 1, if_ = (xc & 1) ? min(in_ + 1, cw - 1) : max(in_ - 1, 0);
        const IN *u0 = row_ptr<IN>(f, 1, jn), *u1 = row_ptr<IN>(f, 1, jf);
        const IN *v0 = row_ptr<IN>(f, 2, jn), *v1 = row_ptr<IN>(f, 2, jf);
        if (left) {
            // co-sited column xc/2 (even xc) or the mean of xc/2 and xc/2+1
            const int i1 = (xc & 1) ? min(in_ + 1, cw - 1) : in_;
            us = 2 * (3 * (load1(u0 + in_) + load1(u0 + i1)) + load1(u1 + in_) + load1(u1 + i1));
            vs = 2 * (3 * (load1(v0 + in_) + load1(v0 + i1)) + load1(v1 + in_) + load1(v1 + i1));
        } else {
            us = 9 * load1(u0 + in_) + 3 * load1(u0 + if_) + 3 * load1(u1 + in_) + load1(u1 + if_);
            vs = 9 * load1(v0 + in_) + 3 * load1(v0 + if_) + 3 * load1(v1 + in_) + load1(v1 + if_);
        }
    } else {
        us = 16 * load1(row_ptr<IN>(f, 1, yc) + xc);
        vs = 16 * load1(row_ptr<IN>(f, 2, yc) + xc);
    }
}

// Packed tensor values of one row of 8 pixels and one channel.
template <typename OUT> struct Row8;
template <> struct Row8<__half> {
    uint4 v;
    __device__ __forceinline__ void set(const float (&x)[kPx])
    {
        v = make_uint4(pack_half2(x[0], x[1]), pack_half2(x[2], x[3]), pack_half2(x[4], x[5]), pack_half2(x[6], x[7]));
    }
    __device__ __forceinline__ void store(__half *p) const
    {
        NNVISR_CHECK_SMEM(p, 16);
        *reinterpret_cast<uint4 *>(p) = v;
    }
    __device__ __forceinline__ void store_n(__half *p, int n) const
    {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < kPx; ++k)
            if (k < n) reinterpret_cast<uint16_t *>(p)[k] = static_cast<uint16_t>(w[k >> 1] >> (16 * (k & 1)));
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
        NNVISR_CHECK_SMEM(p, 32);
        reinterpret_cast<float4 *>(p)[0] = a;
        reinterpret_cast<float4 *>(p)[1] = b;
    }
    __device__ __forceinline__ void store_n(float *p, int n) const
    {
        const float x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int k = 0; k < kPx; ++k)
            if (k < n) p[k] = x[k];
    }
};

// 4 packed tensor values of one chroma row
template <typename OUT> struct Row4;
template <> struct Row4<__half> {
    uint2 v;
    __device__ __forceinline__ void set(const float (&x)[4]) { v = make_uint2(pack_half2(x[0], x[1]), pack_half2(x[2], x[3])); }
    __device__ __forceinline__ void store(__half *p) const
    {
        NNVISR_CHECK_SMEM(p, 8);
        *reinterpret_cast<uint2 *>(p) = v;
    }
    __device__ __forceinline__ void store_n(__half *p, int n) const
    {
        const uint32_t w[2] = {v.x, v.y};
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k < n) reinterpret_cast<uint16_t *>(p)[k] = static_cast<uint16_t>(w[k >> 1] >> (16 * (k & 1)));
    }
};
template <> struct Row4<float> {
    float4 v;
    __device__ __forceinline__ void set(const float (&x)[4]) { v = make_float4(x[0], x[1], x[2], x[3]); }
    __device__ __forceinline__ void store(float *p) const
    {
        NNVISR_CHECK_SMEM(p, 16);
        *reinterpret_cast<float4 *>(p) = v;
    }
    __device__ __forceinline__ void store_n(float *p, int n) const
    {
        const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k < n) p[k] = x[k];
    }
};

// One row of 16x codes -> the three packed channel rows.
template <int FAMILY, typename OUT>
__device__ __forceinline__ void f2t_row(const F2TColour &c, const int (&ys)[kPx], const int (&us)[kPx],
                                        const int (&vs)[kPx], Row8<OUT> (&o)[3])
{
    float R[kPx], G[kPx], B[kPx];
#pragma unroll
    for (int k = 0; k < kPx; ++k) f2t_pixel<FAMILY, OUT>(c, ys[k], us[k], vs[k], R[k], G[k], B[k]);
    o[0].set(R);
    o[1].set(G);
    o[2].set(B);
}

constexpr int kDstRegs = 8;  // destinations of a job held in registers

// Destinations of job j: dst_code[job_dst[j] .. job_dst[j+1]), the first
// kDstRegs in registers.
struct DstList {
    int d0, nd;
    int code[kDstRegs];
    __device__ __forceinline__ void load(const F2TArgs &a, int job)
    {
        d0 = a.job_dst[job];
        nd = a.job_dst[job + 1] - d0;
#pragma unroll
        for (int k = 0; k < kDstRegs; ++k) code[k] = k < nd ? a.dst_code[d0 + k] : 0;
    }
    __device__ __forceinline__ int get(const F2TArgs &a, int d) const
    {
        int cd = 0;
#pragma unroll
        for (int k = 0; k < kDstRegs; ++k)
            if (d == k) cd = code[k];
        if (d >= kDstRegs) cd = a.dst_code[d0 + d];
        return cd;
    }
};

// Store an item's ROWS x 3 packed rows at column x0, row y0 of every
// destination (run, slot) of its frame.
template <int ROWS, typename OUT>
__device__ __forceinline__ void f2t_store(const F2TArgs &a, const DstList &dl, const Row8<OUT> (&out)[ROWS][3], int x0,
                                          int y0)
{
    const int64_t plane = static_cast<int64_t>(a.Hp) * a.Wp;
    const int64_t off = static_cast<int64_t>(y0) * a.Wp + x0;
    const bool vec_store = a.vec_out && (x0 + kPx <= a.Wp);
    const int nvalid = min(kPx, a.Wp - x0);
    for (int d = 0; d < dl.nd; ++d) {
        const int cd = dl.get(a, d);
        OUT *o = reinterpret_cast<OUT *>(a.dst + static_cast<int64_t>(cd >> 5) * a.run_stride +
                                         static_cast<int64_t>(cd & 31) * a.slot_bytes) + off;
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                OUT *q = o + c * plane + static_cast<int64_t>(r) * a.Wp;
                if (vec_store) out[r][c].store(q);
                else out[r][c].store_n(q, nvalid);
            }
        }
    }
}

// t2f job -> (tuple, output slot): dense (job = tuple * M + slot) unless the
// launch skips outputs (NEXT-1 emission), then an explicit code table.
__device__ __forceinline__ void t2f_job(const T2FArgs &a, int job, int &tup, int &o)
{
    if (a.job_code) {
        const int c = a.job_code[job];
        tup = c >> 5;
        o = c & 31;
    } else {
        tup = job / a.M;
        o = job - tup * a.M;
    }
}

// ------------------------------------------------------------ t2f colour
template <typename T> struct T2FConst;
// fp32: ys, yo, cs, co are divided by maxc (see quant)
// yd, yod, csd, co2d: the unnormalised scale / offsets of quant_direct.
template <> struct T2FConst<float> {
    float kr, kb, db, dr, idb, idr, ys, yo, cs, co, maxc, yd, yod, csd, co2d;
    __device__ explicit T2FConst(const T2FColour &c)
        : kr(c.fkr), kb(c.fkb), db(c.fdb), dr(c.fdr), idb(c.fidb), idr(c.fidr), ys(c.fys_n), yo(c.fyo_n),
          cs(c.fcs_n), co(c.fco_n), maxc(c.fmaxc), yd(static_cast<float>(c.ys)), yod(static_cast<float>(c.yo)),
          csd(static_cast<float>(c.cs)), co2d(static_cast<float>(c.co2)) {}
};
template <> struct T2FConst<double> {
    double kr, kb, db, dr, idb, idr, ys, yo, cs, co, maxc, yd, yod, csd, co2d;
    __device__ explicit T2FConst(const T2FColour &c)
        : kr(c.kr), kb(c.kb), db(c.db), dr(c.dr), idb(c.idb), idr(c.idr), ys(c.ys), yo(c.yo), cs(c.cs), co(c.co),
          maxc(c.maxc), yd(c.ys), yod(c.yo), csd(c.cs), co2d(c.co2) {}
};

__device__ __forceinline__ float fma_(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fma_(double a, double b, double c) { return fma(a, b, c); }

// Step B4: clamp to [0, maxc] and round half to even.
// fp32 (8/10-bit codes): q = sat(v * s/maxc + o/maxc) in [0, 1] (FFMA.SAT;
// NaN -> 0), then one FFMA q * maxc + 1.5 * 2^23: the sum lies where the
// spacing of floats is exactly 1, so that single rounding is RNE to an
// integer, which sits in the low mantissa bits (the packers below take only
// the low 16 bits).  fp64 (16-bit codes): a saturating RNE convert to u32 and
// an integer clamp.
__device__ __forceinline__ uint32_t quant(float v, float sn, float on, float maxc)
{
    return __float_as_uint(fmaf(__saturatef(fmaf(v, sn, on)), maxc, 12582912.0f));
}
__device__ __forceinline__ uint32_t quant(double v, double s, double o, double maxc)
{
    // cvt.rni.u32.f64: round half to even, saturating (negative -> 0,
    // NaN -> 0, +inf -> 2^32-1), then the integer clamp to maxc
    return min(__double2uint_rn(fma(v, s, o)), static_cast<uint32_t>(maxc));
}

// Step B4 for tensor values quantised directly (RGB clips, YUV-native
// tensors): q = v * s + o with the unnormalised integer scale / offset in ONE
// FMA.  An fp16 value times s (<= 2^16 - 1) is exact in fp32, so the exact
// .5 ties that fp16 tensors hit often (v on a 2^-11 grid times 219) stay
// ties and round to even as in the oracle; then clamp (fmaxf turns NaN into
// 0) and the magic-add RNE.
__device__ __forceinline__ uint32_t quant_direct(float v, float s, float o, float maxc)
{
    const float q = fminf(fmaxf(fmaf(v, s, o), 0.0f), maxc);
    return __float_as_uint(q + 12582912.0f);
}
__device__ __forceinline__ uint32_t quant_direct(double v, double s, double o, double maxc)
{
    return quant(v, s, o, maxc);
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

__device__ __forceinline__ uint32_t pack4_u8(uint32_t a, uint32_t b, uint32_t c, uint32_t d)
{
    return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}
__device__ __forceinline__ void store_samples8(uint16_t *p, const uint32_t (&v)[kPx])
{
    *reinterpret_cast<uint4 *>(p) = make_uint4(__byte_perm(v[0], v[1], 0x5410), __byte_perm(v[2], v[3], 0x5410),
                                               __byte_perm(v[4], v[5], 0x5410), __byte_perm(v[6], v[7], 0x5410));
}
__device__ __forceinline__ void store_samples8(uint8_t *p, const uint32_t (&v)[kPx])
{
    *reinterpret_cast<uint2 *>(p) = make_uint2(pack4_u8(v[0], v[1], v[2], v[3]), pack4_u8(v[4], v[5], v[6], v[7]));
}
__device__ __forceinline__ void store_samples4(uint16_t *p, const uint32_t (&v)[4])
{
    *reinterpret_cast<uint2 *>(p) = make_uint2(__byte_perm(v[0], v[1], 0x5410), __byte_perm(v[2], v[3], 0x5410));
}
__device__ __forceinline__ void store_samples4(uint8_t *p, const uint32_t (&v)[4])
{
    *reinterpret_cast<uint32_t *>(p) = pack4_u8(v[0], v[1], v[2], v[3]);
}
template <typename OS, int N>
__device__ __forceinline__ void store_samples_n(OS *p, const uint32_t (&v)[N], int n)
{
#pragma unroll
    for (int k = 0; k < N; ++k)
        if (k < n) p[k] = static_cast<OS>(v[k]);
}

// Unpack 8 tensor values of one row and channel.
__device__ __forceinline__ void tunpack8(uint4 v, float (&x)[kPx])
{
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&w[k]));
        x[2 * k] = f.x;
        x[2 * k + 1] = f.y;
    }
}
__device__ __forceinline__ void tunpack8(uint4 a, uint4 b, float (&x)[kPx])
{
    x[0] = __uint_as_float(a.x); x[1] = __uint_as_float(a.y); x[2] = __uint_as_float(a.z); x[3] = __uint_as_float(a.w);
    x[4] = __uint_as_float(b.x); x[5] = __uint_as_float(b.y); x[6] = __uint_as_float(b.z); x[7] = __uint_as_float(b.w);
}
// 8 tensor values from memory (global or shared), 16-byte aligned
__device__ __forceinline__ void tload8(const __half *p, float (&x)[kPx])
{
    NNVISR_CHECK_SMEM(p, 16);
    tunpack8(*reinterpret_cast<const uint4 *>(p), x);
}
__device__ __forceinline__ void tload8(const float *p, float (&x)[kPx])
{
    NNVISR_CHECK_SMEM(p, 32);
    tunpack8(reinterpret_cast<const uint4 *>(p)[0], reinterpret_cast<const uint4 *>(p)[1], x);
}
__device__ __forceinline__ void tload8_stream(const __half *p, float (&x)[kPx]) { tunpack8(ld_stream_v4(p), x); }
__device__ __forceinline__ void tload8_stream(const float *p, float (&x)[kPx])
{
    tunpack8(ld_stream_v4(p), ld_stream_v4(p + 4), x);
}
// 4 tensor values from shared memory (8-byte aligned fp16, 16-byte fp32)
__device__ __forceinline__ void tload4s(const __half *p, float (&x)[4])
{
    NNVISR_CHECK_SMEM(p, 8);
    const uint2 v = *reinterpret_cast<const uint2 *>(p);
    const float2 a = __half22float2(*reinterpret_cast<const __half2 *>(&v.x));
    const float2 b = __half22float2(*reinterpret_cast<const __half2 *>(&v.y));
    x[0] = a.x; x[1] = a.y; x[2] = b.x; x[3] = b.y;
}
__device__ __forceinline__ void tload4s(const float *p, float (&x)[4])
{
    NNVISR_CHECK_SMEM(p, 16);
    const float4 v = *reinterpret_cast<const float4 *>(p);
    x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
}
__device__ __forceinline__ float tload1(const __half *p)
{
    NNVISR_CHECK_SMEM(p, 2);
    return __half2float(p[0]);
}
__device__ __forceinline__ float tload1(const float *p)
{
    NNVISR_CHECK_SMEM(p, 4);
    return p[0];
}

// One output row y (row r of the item) of R', G', B' -> luma codes (and
// 4:4:4 chroma codes, or the 4:2:0 partial 2x2 sums of B-Y', R-Y').
// LEFT (4:2:0 only): the partial sums are the per-row [1,2,1] taps
// (BY[2m-1] + 2 BY[2m]) + BY[2m+1] with BY[-1] = lb (column x0-1, clamped).
template <int FAMILY, typename OS, typename AR, bool LEFT = false>
__device__ __forceinline__ void t2f_row(const T2FConst<AR> &c, const T2FColour &cc, const DevFrame &f, int x0, int y,
                                        int r, const float (&R)[kPx], const float (&G)[kPx], const float (&B)[kPx],
                                        int nvalid, bool vec_store, AR (&sb)[4], AR (&sr)[4], AR lb = AR(0),
                                        AR lr = AR(0))
{
    (void)cc;
    if constexpr (FAMILY == kRGB) {
        uint32_t q[3][kPx];
#pragma unroll
        for (int k = 0; k < kPx; ++k) {
            q[0][k] = quant_direct(static_cast<AR>(R[k]), c.yd, c.yod, c.maxc);
            q[1][k] = quant_direct(static_cast<AR>(G[k]), c.yd, c.yod, c.maxc);
            q[2][k] = quant_direct(static_cast<AR>(B[k]), c.yd, c.yod, c.maxc);
        }
#pragma unroll
        for (int p = 0; p < 3; ++p) {
            OS *out = row_ptr_w<OS>(f, p, y) + x0;
            if (vec_store) store_samples8(out, q[p]);
            else store_samples_n(out, q[p], nvalid);
        }
    } else {
        // Step B2 (luma) + B4: Y' = G + Kr(R-G) + Kb(B-G)
        AR BY[kPx], RY[kPx];
        uint32_t qy[kPx];
        if constexpr (sizeof(AR) == 4) {
            // fp32: pixels 2m, 2m+1 in packed f32x2 (FADD2 / FFMA2: the same
            // per-lane rounding as the scalar FADD / FFMA, half the instructions)
            // pairs A = (0,2), C = (1,3), B = (4,6), D = (5,7): the 4:2:0 column
            // sums BY[2m] + BY[2m+1] of m = 0,1 are then A + C, of m = 2,3 B + D
            const float2 kr2 = make_float2(c.kr, c.kr), kb2 = make_float2(c.kb, c.kb);
            constexpr int P0[4] = {0, 1, 4, 5}, P1[4] = {2, 3, 6, 7};
            float2 by2[4], ry2[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int i0 = P0[q], i1 = P1[q];
                const float2 r2 = make_float2(R[i0], R[i1]), g2 = make_float2(G[i0], G[i1]),
                             b2 = make_float2(B[i0], B[i1]);
                const float2 ng = make_float2(-g2.x, -g2.y);
                const float2 Y2 = __ffma2_rn(kb2, __fadd2_rn(b2, ng), __ffma2_rn(kr2, __fadd2_rn(r2, ng), g2));
                const float2 nY = make_float2(-Y2.x, -Y2.y);
                by2[q] = __fadd2_rn(b2, nY);
                ry2[q] = __fadd2_rn(r2, nY);
                BY[i0] = by2[q].x;
                BY[i1] = by2[q].y;
                RY[i0] = ry2[q].x;
                RY[i1] = ry2[q].y;
                qy[i0] = quant(Y2.x, c.ys, c.yo, c.maxc);
                qy[i1] = quant(Y2.y, c.ys, c.yo, c.maxc);
            }
            if constexpr (FAMILY == kYUV420 && !LEFT) {
                // 4:2:0 centre: ((a+b) + (c+d)) with the row sums (a+b) as A + C, B + D
                const float2 pb01 = __fadd2_rn(by2[0], by2[1]), pb23 = __fadd2_rn(by2[2], by2[3]);
                const float2 pr01 = __fadd2_rn(ry2[0], ry2[1]), pr23 = __fadd2_rn(ry2[2], ry2[3]);
                if (r == 0) {
                    sb[0] = pb01.x; sb[1] = pb01.y; sb[2] = pb23.x; sb[3] = pb23.y;
                    sr[0] = pr01.x; sr[1] = pr01.y; sr[2] = pr23.x; sr[3] = pr23.y;
                } else {
                    const float2 b01 = __fadd2_rn(make_float2(sb[0], sb[1]), pb01), b23 = __fadd2_rn(make_float2(sb[2], sb[3]), pb23);
                    const float2 r01 = __fadd2_rn(make_float2(sr[0], sr[1]), pr01), r23 = __fadd2_rn(make_float2(sr[2], sr[3]), pr23);
                    sb[0] = b01.x; sb[1] = b01.y; sb[2] = b23.x; sb[3] = b23.y;
                    sr[0] = r01.x; sr[1] = r01.y; sr[2] = r23.x; sr[3] = r23.y;
                }
                OS *out = row_ptr_w<OS>(f, 0, y) + x0;
                if (vec_store) store_samples8(out, qy);
                else store_samples_n(out, qy, nvalid);
                return;
            }
        } else {
#pragma unroll
            for (int k = 0; k < kPx; ++k) {
                const AR r_ = R[k], g_ = G[k], b_ = B[k];
                const AR Y = fma_(c.kb, b_ - g_, fma_(c.kr, r_ - g_, g_));
                BY[k] = b_ - Y;
                RY[k] = r_ - Y;
                qy[k] = quant(Y, c.ys, c.yo, c.maxc);
            }
        }
        OS *out = row_ptr_w<OS>(f, 0, y) + x0;
        if (vec_store) store_samples8(out, qy);
        else store_samples_n(out, qy, nvalid);
        if constexpr (FAMILY == kYUV444) {
            uint32_t qb[kPx], qr[kPx];
#pragma unroll
            for (int k = 0; k < kPx; ++k) {
                qb[k] = quant(divide(BY[k], c.db, c.idb), c.cs, c.co, c.maxc);
                qr[k] = quant(divide(RY[k], c.dr, c.idr), c.cs, c.co, c.maxc);
            }
            OS *ob = row_ptr_w<OS>(f, 1, y) + x0, *orr = row_ptr_w<OS>(f, 2, y) + x0;
            if (vec_store) {
                store_samples8(ob, qb);
                store_samples8(orr, qr);
            } else {
                store_samples_n(ob, qb, nvalid);
                store_samples_n(orr, qr, nvalid);
            }
        } else {
            // 4:2:0: accumulate ((a+b) + (c+d)) row by row
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                AR pb, pr;
                if constexpr (LEFT) {
                    const AR b0 = m ? BY[2 * m - 1] : lb, r0 = m ? RY[2 * m - 1] : lr;
                    pb = (b0 + AR(2) * BY[2 * m]) + BY[2 * m + 1];
                    pr = (r0 + AR(2) * RY[2 * m]) + RY[2 * m + 1];
                } else {
                    pb = BY[2 * m] + BY[2 * m + 1];
                    pr = RY[2 * m] + RY[2 * m + 1];
                }
                sb[m] = r == 0 ? pb : sb[m] + pb;
                sr[m] = r == 0 ? pr : sr[m] + pr;
            }
        }
    }
}

// Step B3 + B4 for 4:2:0: 2x2 box mean ((a+b)+(c+d))/4, folded into the
// divisor 4*db (a power-of-two scaling, exact), then quantise and store the
// item's 4 chroma samples of each plane at chroma row y0/2.
// LEFT: the sums carry weight 8 ([1,2,1] per row, two rows): divisor 8*db.
template <typename OS, typename AR, bool LEFT = false>
__device__ __forceinline__ void t2f_chroma420(const T2FConst<AR> &c, const DevFrame &f, int x0, int y0,
                                              const AR (&sb)[4], const AR (&sr)[4], int nvalid, bool vec_store)
{
    constexpr float kW = LEFT ? 8.0f : 4.0f;
    const AR db4 = c.db * AR(kW), dr4 = c.dr * AR(kW), idb4 = c.idb * AR(1.0f / kW), idr4 = c.idr * AR(1.0f / kW);
    uint32_t qb[4], qr[4];
    if constexpr (sizeof(AR) == 4) {
        // packed f32x2 divide (reciprocal product + one FMA correction, as divide())
        auto div2 = [](float2 S, float d, float id) {
            const float2 q0 = __fmul2_rn(S, make_float2(id, id));
            const float2 rr = __ffma2_rn(make_float2(-q0.x, -q0.y), make_float2(d, d), S);
            return __ffma2_rn(rr, make_float2(id, id), q0);
        };
#pragma unroll
        for (int m = 0; m < 4; m += 2) {
            const float2 b2 = div2(make_float2(sb[m], sb[m + 1]), db4, idb4);
            const float2 r2 = div2(make_float2(sr[m], sr[m + 1]), dr4, idr4);
            qb[m] = quant(b2.x, c.cs, c.co, c.maxc);
            qb[m + 1] = quant(b2.y, c.cs, c.co, c.maxc);
            qr[m] = quant(r2.x, c.cs, c.co, c.maxc);
            qr[m + 1] = quant(r2.y, c.cs, c.co, c.maxc);
        }
    } else {
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            qb[m] = quant(divide(sb[m], db4, idb4), c.cs, c.co, c.maxc);
            qr[m] = quant(divide(sr[m], dr4, idr4), c.cs, c.co, c.maxc);
        }
    }
    OS *ob = row_ptr_w<OS>(f, 1, y0 >> 1) + (x0 >> 1), *orr = row_ptr_w<OS>(f, 2, y0 >> 1) + (x0 >> 1);
    if (vec_store) {
        store_samples4(ob, qb);
        store_samples4(orr, qr);
    } else {
        store_samples_n(ob, qb, nvalid / 2);
        store_samples_n(orr, qr, nvalid / 2);
    }
}

}  // namespace dev
}  // namespace nnvisr
