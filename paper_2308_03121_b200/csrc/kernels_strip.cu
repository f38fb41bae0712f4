// kernels_strip.cu -- frames -> tensor for LOW FAN-OUT launches of 4:2:0
// clips: store mode S (each clip frame
// converted once into a frame-major store, §3.3 P:373-382 at batch
// 1), the Fig. 1 batch slots (NEXT-2) and 2-frame windows, where every
// converted frame is written to at most two tensor slots.
//
// There the conversion itself, not HBM, bounds the TMA pipeline of
// kernels_tma.cu (profiles/r01: issue active 56% at 4.0 TB/s in c2 store
// mode, ~35 instructions per pixel, a third of them barrier waits, per-pixel
// branches and address arithmetic).  This kernel is the lean form of the same
// arithmetic:
//
//   * a thread owns 8 luma columns and MARCHES DOWN a band of rows: step k
//     brings chroma row k+1 and emits luma rows 2k+1 (3 x chroma row k + row
//     k+1) and 2k+2 (3 x row k+1 + row k) (reading A5, clamped), so every
//     chroma row is loaded and upsampled once per band, not three times per
//     row pair;
//   * loads are per-thread asynchronous copies (cp.async) kStages steps ahead
//     into shared memory (each thread reads back only its own bytes: no
//     barriers); the chroma halo samples come from the neighbouring lanes by
//     shuffles, at warp edges from a 4-byte copy;
//   * all float work runs on packed f32x2 pairs of pixels {0,2}, {4,6},
//     {1,3}, {5,7}, the pair layout in which the horizontal taps 3*c[m+1] +
//     c[m] / + c[m+2] of adjacent output columns are register pairs, so no
//     operand is shuffled between registers;
//   * stores are 128-bit STGs straight into every destination slot;
//   * the fp16 near-zero test (f2t_fix_tiny) is one vote per 8 pixels, the
//     fp64 recompute only inside that rare branch.
//
// The arithmetic is the TMA fast path's operation for operation (magic-number
// integer->float, exact integer chroma sums -- the horizontal pass first here,
// which gives the same exact integers --, one rounding of Y', one FMA per
// channel), so both kernels give bit-identical tensors (tests/test_gpu_strip.py).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace nnvisr {
namespace {
using namespace dev;

constexpr int kStripThreads = 256;
constexpr int kStages = 4;  // march steps in flight per thread (cp.async)

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

// ---- per-thread asynchronous copies (cp.async, LDGSTS): the loads of the
// next kStages steps wait in shared memory instead of registers.
__device__ __forceinline__ uint32_t smem_addr(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
template <int BYTES>
__device__ __forceinline__ void cp_async(uint32_t dst, const void *src, bool valid)
{
    const int n = valid ? BYTES : 0;  // 0: zero-fill, nothing is read
    if constexpr (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(dst), "l"(src), "n"(BYTES), "r"(n)
                     : "memory");
}
// predicated form: lanes with pred == 0 issue nothing (no branch)
template <int BYTES>
__device__ __forceinline__ void cp_async_if(uint32_t dst, const void *src, bool pred)
{
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q cp.async.ca.shared.global [%0], [%1], %3; }" ::"r"(dst),
                 "l"(src), "r"(static_cast<int>(pred)), "n"(BYTES)
                 : "memory");
}
// predicated 128-bit global stores (no branch)
__device__ __forceinline__ void stg_if(void *p, uint4 v, bool pred)
{
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %5, 0; @q st.global.v4.b32 [%0], {%1, %2, %3, %4}; }" ::"l"(p),
                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(static_cast<int>(pred))
                 : "memory");
}
__device__ __forceinline__ void stg_if(void *p, float4 v, bool pred)
{
    stg_if(p, make_uint4(__float_as_uint(v.x), __float_as_uint(v.y), __float_as_uint(v.z), __float_as_uint(v.w)),
           pred);
}
__device__ __forceinline__ void stg_row_if(__half *p, const Row8<__half> &o, bool pred) { stg_if(p, o.v, pred); }
__device__ __forceinline__ void stg_row_if(float *p, const Row8<float> &o, bool pred)
{
    stg_if(p, o.a, pred);
    stg_if(p + 4, o.b, pred);
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// One pipeline stage = one march step of every thread of the CTA, structure
// of arrays (conflict-free vector reads): luma rows 2k+1, 2k+2 (8 samples
// each), chroma row k+1 of both planes (4 samples each), and per warp the
// 4-byte words holding the warp's outer halo samples (lane 0: i0-1, lane 31:
// i0+4) of both planes.
template <typename IN> struct Stage {
    static constexpr int LB = 8 * sizeof(IN), CB = 4 * sizeof(IN);  // luma / chroma bytes per thread
    __host__ __device__ static constexpr int bytes(int n) { return (n * (2 * LB + 2 * CB) + (n / 32) * 16 + 15) / 16 * 16; }
    // byte offsets inside a stage for thread t of n
    __device__ static int l0(int t) { return t * LB; }
    __device__ static int l1(int t, int n) { return (n + t) * LB; }
    __device__ static int u(int t, int n) { return 2 * n * LB + t * CB; }
    __device__ static int v(int t, int n) { return 2 * n * LB + (n + t) * CB; }
    __device__ static int halo(int w, int n) { return 2 * n * (LB + CB) + 16 * w; }  // [uL, vL, uR, vR]
};

// magic float (2^23 + code) of sample i of packed raw words
__device__ __forceinline__ float magc(uint2 w, int i)  // 16-bit, 4 samples
{
    const uint32_t x = (i < 2) ? w.x : w.y;
    return __uint_as_float(__byte_perm(x, kMagicBits, (i & 1) ? 0x7632 : 0x7610));
}
__device__ __forceinline__ float magc(uint32_t w, int i)  // 8-bit, 4 samples
{
    return __uint_as_float(__byte_perm(w, kMagicBits, 0x7650 + i));
}
template <typename IN> struct Luma;
template <> struct Luma<uint16_t> {  // 8 samples in a uint4
    using V = uint4;
    __device__ static float get(V w, int i)
    {
        const uint32_t x = i < 2 ? w.x : i < 4 ? w.y : i < 6 ? w.z : w.w;
        return __uint_as_float(__byte_perm(x, kMagicBits, (i & 1) ? 0x7632 : 0x7610));
    }
};
template <> struct Luma<uint8_t> {  // 8 samples in a uint2
    using V = uint2;
    __device__ static float get(V w, int i) { return __uint_as_float(__byte_perm(i < 4 ? w.x : w.y, kMagicBits, 0x7650 + (i & 3))); }
};
// halo samples inside their aligned 4-byte words: the left word ends at
// sample i0-1, the right word starts at sample i0+4
template <typename IN> __device__ __forceinline__ float halo_l(uint32_t w)
{
    return __uint_as_float(kMagicBits | (sizeof(IN) == 2 ? (w >> 16) : (w >> 24)));
}
template <typename IN> __device__ __forceinline__ float halo_r(uint32_t w)
{
    return __uint_as_float(kMagicBits | (sizeof(IN) == 2 ? (w & 0xffffu) : (w & 0xffu)));
}

// A horizontally upsampled chroma row of the thread's 8 columns, 4x scale
// minus the offset, in the pixel-pair layout A = {0,2}, B = {4,6},
// C = {1,3}, D = {5,7}.
struct HRow {
    float2 A, B, C, D;
};

// Chroma row from its 4 own raw samples (halos by shuffles / edge words,
// clamped at the plane edges): centre siting 3*c[m+1] + c[m] (even column
// 2m) / + c[m+2] (odd 2m+1); LEFT (MPEG-2) 4*c[m+1] / 2*(c[m+1] + c[m+2])
// (reading A5).  Every lane of the warp calls it (shuffles).
template <typename IN, bool LEFT>
__device__ __forceinline__ HRow chroma_row(typename Pack<IN>::V4 own, uint32_t hl, uint32_t hr, bool lane0,
                                           bool lane31, bool has_l, bool has_r, float coff)
{
    const float c1 = magc(own, 0), c2 = magc(own, 1), c3 = magc(own, 2), c4 = magc(own, 3);
    const float up = __shfl_up_sync(0xffffffffu, c4, 1), dn = __shfl_down_sync(0xffffffffu, c1, 1);
    float c0 = lane0 ? halo_l<IN>(hl) : up;
    float c5 = lane31 ? halo_r<IN>(hr) : dn;
    c0 = has_l ? c0 : c1;
    c5 = has_r ? c5 : c4;
    const float2 o2 = f2(-coff, -coff);
    const float2 E01 = fadd2(f2(c0, c1), o2), E23 = fadd2(f2(c2, c3), o2), E45 = fadd2(f2(c4, c5), o2);
    const float2 O12 = f2(E01.y, E23.x), O34 = f2(E23.y, E45.x);
    HRow h;
    if constexpr (!LEFT) {
        const float2 k3 = f2(3.0f, 3.0f);
        h.A = ffma2(k3, O12, E01);  // pixels 0, 2: 3c1 + c0, 3c2 + c1
        h.B = ffma2(k3, O34, E23);  // 4, 6: 3c3 + c2, 3c4 + c3
        h.C = ffma2(k3, O12, E23);  // 1, 3: 3c1 + c2, 3c2 + c3
        h.D = ffma2(k3, O34, E45);  // 5, 7: 3c3 + c4, 3c4 + c5
    } else {
        const float2 k4 = f2(4.0f, 4.0f), k2 = f2(2.0f, 2.0f);
        h.A = fmul2(k4, O12);
        h.B = fmul2(k4, O34);
        h.C = fmul2(k2, fadd2(O12, E23));
        h.D = fmul2(k2, fadd2(O34, E45));
    }
    return h;
}

// fp16 near-zero values of a row recomputed in fp64 (f2t_fix_tiny).  (Out
// of line -- __noinline__ -- it costs a 576-byte stack frame and 3x the
// kernel time on B200: inlined.)
__device__ __forceinline__ void fix_tiny_row(const F2TColour &col, const float2 (&dy)[4], const float2 (&du)[4],
                                          const float2 (&dv)[4], float2 (&R)[4], float2 (&G)[4], float2 (&B)[4])
{
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        f2t_fix_tiny<__half>(col, dy[p].x, du[p].x, dv[p].x, R[p].x, G[p].x, B[p].x);
        f2t_fix_tiny<__half>(col, dy[p].y, du[p].y, dv[p].y, R[p].y, G[p].y, B[p].y);
    }
}

// One luma row of 8 pixels: chroma 3*near + far (16x scale minus the
// offset, exact), Y' = (code - y_off/16) * 16 y_scale (one rounding), one
// FMA per channel; fp16 near-zero values recomputed in fp64 (rare branch).
template <typename IN, typename OUT>
__device__ __forceinline__ void convert_row(const F2TColour &col, typename Luma<IN>::V lraw, const HRow &nu,
                                            const HRow &fu, const HRow &nv, const HRow &fv, Row8<OUT> (&o)[3])
{
    const float2 k3 = f2(3.0f, 3.0f);
    float2 du[4], dv[4], dy[4], Y[4];
    du[0] = ffma2(k3, nu.A, fu.A);
    du[1] = ffma2(k3, nu.B, fu.B);
    du[2] = ffma2(k3, nu.C, fu.C);
    du[3] = ffma2(k3, nu.D, fu.D);
    dv[0] = ffma2(k3, nv.A, fv.A);
    dv[1] = ffma2(k3, nv.B, fv.B);
    dv[2] = ffma2(k3, nv.C, fv.C);
    dv[3] = ffma2(k3, nv.D, fv.D);
    const float yoff = kMagic + static_cast<float>(col.y_off >> 4);
    const float ys16 = 16.0f * col.y_scale;
    const float2 yo2 = f2(-yoff, -yoff), ys2 = f2(ys16, ys16);
    // pair p holds pixels (P0[p], P1[p]): A = {0,2}, B = {4,6}, C = {1,3}, D = {5,7}
    constexpr int P0[4] = {0, 4, 1, 5}, P1[4] = {2, 6, 3, 7};
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        dy[p] = fadd2(f2(Luma<IN>::get(lraw, P0[p]), Luma<IN>::get(lraw, P1[p])), yo2);
        Y[p] = fmul2(dy[p], ys2);
    }
    const float2 rv2 = f2(col.r_v, col.r_v), bu2 = f2(col.b_u, col.b_u);
    const float2 gu2 = f2(-col.g_u, -col.g_u), gv2 = f2(-col.g_v, -col.g_v);
    float2 R[4], G[4], B[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        R[p] = ffma2(rv2, dv[p], Y[p]);
        B[p] = ffma2(bu2, du[p], Y[p]);
        G[p] = ffma2(gv2, dv[p], ffma2(gu2, du[p], Y[p]));
    }
    if constexpr (sizeof(OUT) == 2) {
        float mn = 1.0f;
#pragma unroll
        for (int p = 0; p < 4; ++p)
            mn = fminf(mn, fminf(fminf(fminf(fabsf(R[p].x), fabsf(R[p].y)), fminf(fabsf(G[p].x), fabsf(G[p].y))),
                                 fminf(fabsf(B[p].x), fabsf(B[p].y))));
        if (mn < kF16Tiny) fix_tiny_row(col, dy, du, dv, R, G, B);  // rare: the fp64 near-zero recompute
        // pixels (0,1) = (A.x, C.x), (2,3) = (A.y, C.y), (4,5) = (B.x, D.x), (6,7) = (B.y, D.y)
        o[0].v = make_uint4(pack_half2(R[0].x, R[2].x), pack_half2(R[0].y, R[2].y), pack_half2(R[1].x, R[3].x),
                            pack_half2(R[1].y, R[3].y));
        o[1].v = make_uint4(pack_half2(G[0].x, G[2].x), pack_half2(G[0].y, G[2].y), pack_half2(G[1].x, G[3].x),
                            pack_half2(G[1].y, G[3].y));
        o[2].v = make_uint4(pack_half2(B[0].x, B[2].x), pack_half2(B[0].y, B[2].y), pack_half2(B[1].x, B[3].x),
                            pack_half2(B[1].y, B[3].y));
    } else {
        o[0].a = make_float4(R[0].x, R[2].x, R[0].y, R[2].y);
        o[0].b = make_float4(R[1].x, R[3].x, R[1].y, R[3].y);
        o[1].a = make_float4(G[0].x, G[2].x, G[0].y, G[2].y);
        o[1].b = make_float4(G[1].x, G[3].x, G[1].y, G[3].y);
        o[2].a = make_float4(B[0].x, B[2].x, B[0].y, B[2].y);
        o[2].b = make_float4(B[1].x, B[3].x, B[1].y, B[3].y);
    }
}

// Store one row (3 channels) at tensor row y, column x of every destination.
template <typename OUT>
__device__ __forceinline__ void store_row(const F2TArgs &a, const DstList &dl, const Row8<OUT> (&o)[3], int x, int y)
{
    const int64_t plane = static_cast<int64_t>(a.Hp) * a.Wp;
    const int64_t off = static_cast<int64_t>(y) * a.Wp + x;
    for (int d = 0; d < dl.nd; ++d) {
        const int cd = dl.get(a, d);
        OUT *q = reinterpret_cast<OUT *>(a.dst + static_cast<int64_t>(cd >> 5) * a.run_stride +
                                         static_cast<int64_t>(cd & 31) * a.slot_bytes) + off;
#pragma unroll
        for (int c = 0; c < 3; ++c) o[c].store(q + c * plane);
    }
}

// Destination rows of one tile, walked row by row: ND = 1 or 2 slots held as
// pointers (one add per row and slot), ND = 0 any number (through dl).
template <typename OUT, int ND> struct DstRows {
    char *q[ND];
    int64_t plane_b;
    int64_t row_b;
#ifdef NNVISR_CHECKED
    const char *lo[ND];  // checked builds: every store lands inside its (run, slot)
    int64_t slot_b;
#endif
    __device__ __forceinline__ void init(const F2TArgs &a, const DstList &dl, int x, int y)
    {
        plane_b = static_cast<int64_t>(a.Hp) * a.Wp * sizeof(OUT);
        row_b = static_cast<int64_t>(a.Wp) * sizeof(OUT);
#pragma unroll
        for (int d = 0; d < ND; ++d) {
            const int cd = dl.code[d];
            q[d] = a.dst + static_cast<int64_t>(cd >> 5) * a.run_stride + static_cast<int64_t>(cd & 31) * a.slot_bytes +
                   (static_cast<int64_t>(y) * a.Wp + x) * static_cast<int64_t>(sizeof(OUT));
#ifdef NNVISR_CHECKED
            lo[d] = a.dst + static_cast<int64_t>(cd >> 5) * a.run_stride + static_cast<int64_t>(cd & 31) * a.slot_bytes;
            slot_b = a.slot_bytes;
#endif
        }
    }
    __device__ __forceinline__ void put(const Row8<OUT> (&o)[3], bool pred)
    {
#pragma unroll
        for (int d = 0; d < ND; ++d) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
#ifdef NNVISR_CHECKED
                NNVISR_CHECK(!pred || (q[d] + c * plane_b >= lo[d] &&
                                       q[d] + c * plane_b + kPx * sizeof(OUT) <= lo[d] + slot_b));
#endif
                stg_row_if(reinterpret_cast<OUT *>(q[d] + c * plane_b), o[c], pred);
            }
            q[d] += row_b;
        }
    }
    __device__ __forceinline__ void skip()
    {
#pragma unroll
        for (int d = 0; d < ND; ++d) q[d] += row_b;
    }
};
template <typename OUT> struct DstRows<OUT, 0> {
    const F2TArgs *a;
    const DstList *dl;
    int x, y;
    __device__ __forceinline__ void init(const F2TArgs &a_, const DstList &dl_, int x_, int y_)
    {
        a = &a_;
        dl = &dl_;
        x = x_;
        y = y_;
    }
    __device__ __forceinline__ void put(const Row8<OUT> (&o)[3], bool pred)
    {
        if (pred) store_row<OUT>(*a, *dl, o, x, y);
        ++y;
    }
    __device__ __forceinline__ void skip() { ++y; }
};

// Ragged right edge / padding columns: per-sample clamped taps (integer path).
template <typename IN, typename OUT>
__device__ __forceinline__ void slow_row(const F2TArgs &a, const DstList &dl, const DevFrame &f, int x, int y)
{
    int ys[kPx], us[kPx], vs[kPx];
#pragma unroll
    for (int k = 0; k < kPx; ++k) f2t_codes_scalar<kYUV420, IN>(f, a.W, a.H, x + k, y, ys[k], us[k], vs[k], a.left);
    Row8<OUT> o[3];
    f2t_row<kYUV420, OUT>(a.col, ys, us, vs, o);
    const int64_t plane = static_cast<int64_t>(a.Hp) * a.Wp;
    const int64_t off = static_cast<int64_t>(y) * a.Wp + x;
    const int n = min(kPx, a.Wp - x);
    for (int d = 0; d < dl.nd; ++d) {
        const int cd = dl.get(a, d);
        OUT *q = reinterpret_cast<OUT *>(a.dst + static_cast<int64_t>(cd >> 5) * a.run_stride +
                                         static_cast<int64_t>(cd & 31) * a.slot_bytes) + off;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (n == kPx) o[c].store(q + c * plane);
            else o[c].store_n(q + c * plane, n);
        }
    }
}

// Chroma row j of this thread read directly (band prologue, padding rows).
template <typename IN, bool LEFT>
__device__ __forceinline__ HRow chroma_row_direct(const char *ub, int64_t pitch, int j, bool live, bool lane0,
                                                  bool lane31, bool has_l, bool has_r, float coff)
{
    using V4 = typename Pack<IN>::V4;
    const IN *u = reinterpret_cast<const IN *>(ub + j * pitch);
    const V4 r = live ? *reinterpret_cast<const V4 *>(u) : V4{};
    const uint32_t sh = sizeof(IN) == 2 ? 16 : 24;
    const uint32_t hl = (lane0 && has_l && live) ? static_cast<uint32_t>(load1(u - 1)) << sh : 0u;
    const uint32_t hr = (lane31 && has_r && live) ? static_cast<uint32_t>(load1(u + 4)) : 0u;
    return chroma_row<IN, LEFT>(r, hl, hr, lane0, lane31, has_l, has_r, coff);
}

// Rows [y0, y1) of a band for the 8 columns at x of every thread of the CTA
// (a strip of 8 x blockDim.x columns).  Step s (s = 0 .. steps-1) brings
// chroma row y0/2 + s and luma rows y0 + 2s - 1 (s >= 1), y0 + 2s (< the
// band's last real row) through the cp.async ring; padding rows (y >= H)
// replicate row H-1.  Lanes whose columns are not all inside the frame run
// along on dummy data (their shuffles are needed) and are converted by the
// scalar path afterwards; lanes past the padded width store nothing.
template <typename IN, typename OUT, bool LEFT, class Dst>
__device__ __forceinline__ void march(const F2TArgs &a, const DevFrame &f, int x, int y0, int y1, Dst &dst,
                                      uint8_t *smem)
{
    using V4 = typename Pack<IN>::V4;
    using LV = typename Luma<IN>::V;
    using S = Stage<IN>;
    const int n = blockDim.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int cw = a.W >> 1, ch = a.H >> 1, i0 = x >> 1;
    // rd: loads inside the rows (x < W; padding columns read nothing);
    // live: a tensor column (stores)
    const bool rd = x < a.W, live = x < a.Wp;
    const bool has_l = i0 > 0, has_r = i0 + 4 < cw, lane0 = lane == 0, lane31 = lane == 31;
    const float coff = kMagic + static_cast<float>(a.col.c_off >> 4);
    const int64_t lp = f.pitch[0], up = f.pitch[1], vp = f.pitch[2];
    const char *lbase = static_cast<const char *>(f.plane[0]) + x * sizeof(IN);
    const char *ub = static_cast<const char *>(f.plane[1]) + i0 * sizeof(IN);
    const char *vb = static_cast<const char *>(f.plane[2]) + i0 * sizeof(IN);
    const int SB = S::bytes(n);
    const uint32_t sbase = smem_addr(smem);
    const int yr1 = min(y1, a.H);
    const int steps = yr1 > y0 ? (yr1 - y0) / 2 + 1 : 0;
    if (steps > 0) {
        // ring entry r: r = 0 the band's first far chroma row y0/2 - 1
        // (clamped), r = s + 1 step s; running source pointers of the next
        // entry to issue
        const char *la = lbase + static_cast<int64_t>(y0 - 3) * lp;  // luma row y0 + 2s - 1 (entry r: y0 + 2r - 3)
        const char *lb = lbase + static_cast<int64_t>(y0 - 2) * lp;  // luma row y0 + 2s
        int jn = y0 / 2 - 1;                                         // chroma row of the next entry (unclamped)
        const int hoff = lane0 ? -4 : 4 * static_cast<int>(sizeof(IN));  // aligned halo words (lanes 0 / 31)
        const bool hv = rd && (lane0 ? has_l : has_r) && (lane0 || lane31);
        const uint32_t ol0 = S::l0(t), ol1 = S::l1(t, n), ou = S::u(t, n), ov = S::v(t, n), oh = S::halo(w, n);
        const uint32_t oh_mine = oh + (lane31 ? 8 : 0);
        int ri = 0;  // next ring entry to issue
        auto issue = [&]() {
            const uint32_t st = sbase + (ri & (kStages - 1)) * SB;
            const bool in = rd && ri <= steps;
            const int jc = min(max(jn, 0), ch - 1);
            const char *un = ub + static_cast<int64_t>(jc) * up, *vn = vb + static_cast<int64_t>(jc) * vp;
#ifdef NNVISR_CHECKED
            {  // every copy lands in this stage and reads inside its plane
                const uint32_t e = st + SB;
                NNVISR_CHECK(st + ol0 + S::LB <= e && st + ol1 + S::LB <= e && st + ou + S::CB <= e && st + ov + S::CB <= e &&
                             st + oh_mine + 8 <= e && sbase + kStages * SB <= sbase + (uint32_t)(kStages * SB));
                auto inside = [&](const char *p, int n, int pl, int rows) {
                    const char *b = static_cast<const char *>(f.plane[pl]);
                    return p >= b && p + n <= b + rows * f.pitch[pl];
                };
                NNVISR_CHECK(!(in && ri >= 2) || inside(la, S::LB, 0, a.H));
                NNVISR_CHECK(!(in && ri >= 1 && ri < steps) || inside(lb, S::LB, 0, a.H));
                NNVISR_CHECK(!in || (inside(un, S::CB, 1, ch) && inside(vn, S::CB, 2, ch)));
                NNVISR_CHECK(!(in && hv) || (inside(un + hoff, 4, 1, ch) && inside(vn + hoff, 4, 2, ch)));
            }
#endif
            cp_async<S::LB>(st + ol0, la, in && ri >= 2);
            cp_async<S::LB>(st + ol1, lb, in && ri >= 1 && ri < steps);
            cp_async<S::CB>(st + ou, un, in);
            cp_async<S::CB>(st + ov, vn, in);
            cp_async_if<4>(st + oh_mine, un + hoff, in && hv);
            cp_async_if<4>(st + oh_mine + 4, vn + hoff, in && hv);
            cp_commit();
            la += 2 * lp;
            lb += 2 * lp;
            ++jn;
            ++ri;
        };
#pragma unroll
        for (int k = 0; k < kStages - 1; ++k) issue();
        // entry 0: chroma row y0/2 - 1 (clamped), the far row of the band's first luma row
        auto chroma_entry = [&](int r, HRow &wu, HRow &wv) {
            const uint8_t *st = smem + (r & (kStages - 1)) * SB;
            const uint32_t *hw = reinterpret_cast<const uint32_t *>(st + oh);
            wu = chroma_row<IN, LEFT>(*reinterpret_cast<const V4 *>(st + ou), hw[0], hw[2], lane0, lane31, has_l,
                                      has_r, coff);
            wv = chroma_row<IN, LEFT>(*reinterpret_cast<const V4 *>(st + ov), hw[1], hw[3], lane0, lane31, has_l,
                                      has_r, coff);
            return st;
        };
        HRow bu, bv;
        issue();
        cp_wait<kStages - 1>();
        chroma_entry(0, bu, bv);
        HRow cu, cv;
        // step s: chroma row y0/2 + s arrives in (wu, wv); rows y0 + 2s - 1
        // (near = previous row p, far = w; not at s = 0) and y0 + 2s (near w,
        // far p; not at the last step)
        auto step = [&](int s, HRow &pu, HRow &pv, HRow &wu, HRow &wv, bool first_row, bool second_row) {
            issue();
            cp_wait<kStages - 1>();
            const uint8_t *st = chroma_entry(s + 1, wu, wv);
            Row8<OUT> o[3];
            if (first_row) {
                convert_row<IN, OUT>(a.col, *reinterpret_cast<const LV *>(st + ol0), pu, wu, pv, wv, o);
                dst.put(o, live);
            }
            if (second_row) {
                convert_row<IN, OUT>(a.col, *reinterpret_cast<const LV *>(st + ol1), wu, pu, wv, pv, o);
                dst.put(o, live);
            }
        };
        // steps >= 2; even steps hold (p, w) = (b, c), odd ones (c, b)
        for (int s = 0; s < steps; s += 2) {
            step(s, bu, bv, cu, cv, s >= 1, s + 1 < steps);
            if (s + 1 >= steps) break;
            step(s + 1, cu, cv, bu, bv, true, s + 2 < steps);
        }
        cp_wait<0>();
    }
    // padding rows (y >= H, reading A6): row H-1 (near = far = chroma row ch-1)
    if (y1 > a.H) {
        const HRow pu = chroma_row_direct<IN, LEFT>(ub, up, ch - 1, rd, lane0, lane31, has_l, has_r, coff);
        const HRow pv = chroma_row_direct<IN, LEFT>(vb, vp, ch - 1, rd, lane0, lane31, has_l, has_r, coff);
        // every lane converts (lanes outside the frame convert zeros; ragged
        // ones are redone by the scalar path), live lanes store
        const LV l = rd ? *reinterpret_cast<const LV *>(lbase + static_cast<int64_t>(a.H - 1) * lp) : LV{};
        Row8<OUT> o[3];
        convert_row<IN, OUT>(a.col, l, pu, pu, pv, pv, o);
        for (int y = max(y0, a.H); y < y1; ++y) dst.put(o, live);
    }
}

// Tile = (job, band of a.band luma rows, strip of 8 x blockDim.x columns).
// Every thread of a CTA walks the same tiles (warp-uniform loops: the march
// shuffles chroma halos between lanes).
template <typename IN, typename OUT, bool LEFT>
__global__ void __launch_bounds__(kStripThreads, 2) f2t_strip420(const F2TArgs a)
{
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int64_t next_tile;
    const int bands = (a.Hp + a.band - 1) / a.band;
    const int64_t per_job = static_cast<int64_t>(bands) * a.nseg;
    // persistent CTAs, dynamic tiles: each CTA takes the launch's next tile
    // from the zeroed per-launch counter, so fast SMs take more tiles and no
    // SM idles through a long static share (r02 ncu: SMs active 86% of the
    // kernel with static striding)
    for (int64_t iter = 0;; ++iter) {
        if (threadIdx.x == 0)  // (no counter: static tiles b, b + G, ...)
            next_tile = a.tile_counter ? static_cast<int64_t>(atomicAdd(a.tile_counter, 1ull))
                                       : blockIdx.x + iter * gridDim.x;
        __syncthreads();
        const int64_t t = next_tile;
        __syncthreads();
        if (t >= a.tiles) break;
        const int job = static_cast<int>(t / per_job);
        const int rem = static_cast<int>(t - job * per_job);
        const int band = rem / a.nseg, strip = rem - band * a.nseg;
        const int x = (strip * blockDim.x + threadIdx.x) * kPx;
        const DevFrame f = load_frame(a.frames + a.job_frame[job]);
        DstList dl;
        dl.load(a, job);
        const int y0 = band * a.band, y1 = min(y0 + a.band, a.Hp);
        if (dl.nd == 1) {
            DstRows<OUT, 1> d;
            d.init(a, dl, x, y0);
            march<IN, OUT, LEFT>(a, f, x, y0, y1, d, smem);
        } else if (dl.nd == 2) {
            DstRows<OUT, 2> d;
            d.init(a, dl, x, y0);
            march<IN, OUT, LEFT>(a, f, x, y0, y1, d, smem);
        } else {
            DstRows<OUT, 0> d;
            d.init(a, dl, x, y0);
            march<IN, OUT, LEFT>(a, f, x, y0, y1, d, smem);
        }
        if (x < a.Wp && x + kPx > a.W) {  // ragged right edge / padding columns: scalar path
            for (int y = y0; y < y1; ++y) slow_row<IN, OUT>(a, dl, f, x, y);
        }
        __syncwarp();
    }
}

template <typename IN, typename OUT, bool LEFT>
cudaError_t launch(F2TArgs a, cudaStream_t s)
{
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    // columns: strips of 8 x threads (threads = the row's 8-column groups,
    // whole warps, <= 256); rows: bands of a.band luma rows (even)
    const int groups = a.Wp / kPx;
    a.nseg = (groups + kStripThreads - 1) / kStripThreads;
    const int threads = ((groups + a.nseg - 1) / a.nseg + 31) / 32 * 32;  // equal strips, whole warps
    auto kernel = f2t_strip420<IN, OUT, LEFT>;
    const int smem = kStages * Stage<IN>::bytes(threads);
    cudaError_t err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    if (err != cudaSuccess) return err;
    const int64_t slots = static_cast<int64_t>(sms) * std::max(per_sm, 1);
    // bands: ~NNVISR_F2T_STRIP_TPC (default 12) tiles per resident CTA, so
    // the dynamic schedule's tail is short, and at least 32 rows (each tile
    // start waits one memory latency before its ring fills)
    const char *e = std::getenv("NNVISR_F2T_STRIP_ROWS");
    const char *tpc_e = std::getenv("NNVISR_F2T_STRIP_TPC");
    const int64_t tpc = tpc_e && *tpc_e ? std::max(1, std::atoi(tpc_e)) : 12;
    const int64_t rows_all = static_cast<int64_t>(a.Hp) * a.jobs * a.nseg;
    const int64_t auto_band = std::max<int64_t>(32, std::min<int64_t>(a.Hp, rows_all / (tpc * slots)));
    a.band = e && *e ? std::max(2, std::atoi(e) & ~1) : static_cast<int>(auto_band + 1) & ~1;
    const int bands = (a.Hp + a.band - 1) / a.band;
    a.tiles = a.jobs * bands * a.nseg;
    if (a.tiles <= 0) return cudaSuccess;
    const int64_t grid = std::min<int64_t>(a.tiles, slots);
    kernel<<<static_cast<int>(grid), threads, smem, s>>>(a);
    return cudaGetLastError();
}

template <typename IN, typename OUT>
cudaError_t launch_sited(const F2TArgs &a, cudaStream_t s)
{
    return a.left ? launch<IN, OUT, true>(a, s) : launch<IN, OUT, false>(a, s);
}

}  // namespace

// 4:2:0 RGB tensors with 16-byte aligned planes, pitches and tensor rows
// (the caller checked a.tma_ok).
cudaError_t launch_f2t_strip(int bits, int dtype, const F2TArgs &a, cudaStream_t s)
{
    if (bits == 8) return dtype == kF16 ? launch_sited<uint8_t, __half>(a, s) : launch_sited<uint8_t, float>(a, s);
    return dtype == kF16 ? launch_sited<uint16_t, __half>(a, s) : launch_sited<uint16_t, float>(a, s);
}

}  // namespace nnvisr
