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
//   * loads are per-thread asynchronous copies (cp.async) into a ring of
//     shared-memory stages laid out at compile time; each lane reads its
//     own luma and chroma bytes and its neighbouring lanes' outer chroma
//     samples (one warp barrier per step), the warp's outer halo words are
//     copied by lanes 0 and 31 into pads around the warp's block;
//   * all float work runs on packed f32x2 pairs of pixels {0,7}, {1,2},
//     {3,4}, {5,6}: the centre horizontal taps of {1,2} and {5,6} are
//     3 x (a natural sample pair) + that pair swapped (an operand swizzle,
//     no register moves), {0,7} and {3,4} two scalar FMAs each;
//   * 16-bit samples become magic floats with one LOP3 / LEA.HI each;
//   * stores are 128-bit STGs straight into every destination slot,
//     addressed with 32-bit plane / row offsets;
//   * the fp16 near-zero test (f2t_fix_tiny) is one vote per 8 pixels on the
//     packed row; the rare branch recomputes the row from its inputs (nothing
//     but the packed row stays live across the test);
//   * persistent CTAs take tiles from a per-launch counter, the next index
//     fetched while the current tile runs.
//
// r02 B200 measurements (tools/ab_r02s.sh, tools/ab_cfg.sh): the rewrite
// executes 13% fewer instructions (ncu 243 M vs 280 M per c5
// region fill) at the same time (c2 / c5 store 5.3 / 5.45 TB/s, c4 8-bit
// Fig. 1 batches 4.7 vs 5.0): the kernel is bound by the memory-level
// parallelism of 16 warps per SM (128 registers) on a 1-read : 2-write mix,
// not by issue (a 1:2 streaming probe reaches 5.8 TB/s at 32 warps per SM,
// 6.25 at 64; tools/hbm_probe.cu).
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
#ifndef NNVISR_STRIP_MINB
#define NNVISR_STRIP_MINB 2  // resident CTAs per SM the register budget is cut for
#endif
#ifndef NNVISR_STRIP_LAYOUT_THREADS
#define NNVISR_STRIP_LAYOUT_THREADS kStripThreads
#endif
#ifndef NNVISR_STRIP_STAGES
#define NNVISR_STRIP_STAGES 4
#endif
// ring entries per thread (cp.async): kStages - 2 steps ahead at each wait
constexpr int kStages = NNVISR_STRIP_STAGES;

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

// One pipeline stage = one march step of every thread of the CTA, laid out
// for kStripThreads threads at compile time (constant offsets: no address
// arithmetic from blockDim per step): luma rows 2k+1, 2k+2 (8 samples per
// thread each, thread-major), then chroma row k+1 of U and of V in per-warp
// blocks [pad | 32 lanes x 4 samples | pad].  Lane l reads its neighbours'
// outer samples (the word before its own samples, the word after) from the
// block after a __syncwarp; the pads hold the warp's outer halo words,
// copied by lanes 0 and 31 (i0-1 in the pad's last word, i0+4 in the right
// pad's first word), so every lane reads the same way.
template <typename IN> struct Stage {
    static constexpr int LB = 8 * sizeof(IN), CB = 4 * sizeof(IN);  // luma / chroma bytes per thread
    static constexpr int HB = CB;                                   // pad per side (own samples stay CB-aligned)
    static constexpr int WB = 32 * CB + 2 * HB;                     // chroma bytes per warp block
    static constexpr int kT = NNVISR_STRIP_LAYOUT_THREADS;  // threads the layout is cut for
    static constexpr int kWarps = kT / 32;
    static constexpr int kL0 = 0, kL1 = kT * LB;
    static constexpr int kU = 2 * kT * LB, kV = kU + kWarps * WB;
    static constexpr int kBytes = (kV + kWarps * WB + 127) / 128 * 128;
    __device__ static int own_c(int t) { return (t >> 5) * WB + HB + (t & 31) * CB; }
};

// magic float (2^23 + code) of sample i of packed raw words
// 16-bit sample h (0 low, 1 high) of a word as a magic float: one LOP3 / LEA.HI
__device__ __forceinline__ float mag16(uint32_t x, int h)
{
    if (h) return __uint_as_float((x >> 16) | kMagicBits);
    uint32_t r;  // (x & 0xffff) | magic in one LOP3 (the magic in a register)
    asm("lop3.b32 %0, %1, 0xffff, %2, 0xEA;" : "=r"(r) : "r"(x), "r"(kMagicBits));
    return __uint_as_float(r);
}
__device__ __forceinline__ float magc(uint2 w, int i)  // 16-bit, 4 samples
{
    return mag16(i < 2 ? w.x : w.y, i & 1);
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
        return mag16(i < 2 ? w.x : i < 4 ? w.y : i < 6 ? w.z : w.w, i & 1);
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
// minus the offset, in the pixel-pair layout A = {0,7}, B = {1,2},
// C = {3,4}, D = {5,6}: B and D are 3 x (a natural sample pair) + the same
// pair swapped, so the centre taps need no operand moved between registers.
struct HRow {
    float2 A, B, C, D;
};
// pair p of a row holds pixels (kP0[p], kP1[p])
__device__ constexpr int kP0[4] = {0, 1, 3, 5}, kP1[4] = {7, 2, 4, 6};

// Horizontal taps of one chroma row from samples c0 .. c5 (magic floats;
// c0 = i0-1, c5 = i0+4, already clamped): centre siting 3*c[m+1] + c[m]
// (even column 2m) / + c[m+2] (odd 2m+1); LEFT (MPEG-2) 4*c[m+1] /
// 2*(c[m+1] + c[m+2]) (reading A5).  Exact integers throughout.
template <bool LEFT>
__device__ __forceinline__ HRow chroma_taps(float c0, float c1, float c2, float c3, float c4, float c5, float coff)
{
    const float2 o2 = f2(-coff, -coff);
    const float2 P = fadd2(f2(c1, c2), o2), Q = fadd2(f2(c3, c4), o2), H = fadd2(f2(c0, c5), o2);
    HRow h;
    if constexpr (!LEFT) {
        const float2 k3 = f2(3.0f, 3.0f);
        h.A = f2(fmaf(3.0f, P.x, H.x), fmaf(3.0f, Q.y, H.y));  // pixels 0, 7: 3c1 + c0, 3c4 + c5
        h.B = ffma2(k3, P, f2(P.y, P.x));                       // 1, 2: 3c1 + c2, 3c2 + c1
        h.C = f2(fmaf(3.0f, P.y, Q.x), fmaf(3.0f, Q.x, P.y));  // 3, 4: 3c2 + c3, 3c3 + c2
        h.D = ffma2(k3, Q, f2(Q.y, Q.x));                       // 5, 6: 3c3 + c4, 3c4 + c3
    } else {
        h.A = f2(4.0f * P.x, 2.0f * (Q.y + H.y));  // 0: 4c1, 7: 2(c4 + c5)
        h.B = f2(2.0f * (P.x + P.y), 4.0f * P.y);  // 1: 2(c1 + c2), 2: 4c2
        h.C = f2(2.0f * (P.y + Q.x), 4.0f * Q.x);  // 3: 2(c2 + c3), 4: 4c3
        h.D = f2(2.0f * (Q.x + Q.y), 4.0f * Q.y);  // 5: 2(c3 + c4), 6: 4c4
    }
    return h;
}

// Chroma row from its 4 own raw samples and the words before / after them
// (hl ends at sample i0-1, hr starts at i0+4), clamped at the plane edges.
template <typename IN, bool LEFT>
__device__ __forceinline__ HRow chroma_row(typename Pack<IN>::V4 own, uint32_t hl, uint32_t hr, bool has_l, bool has_r,
                                           float coff)
{
    const float c1 = magc(own, 0), c2 = magc(own, 1), c3 = magc(own, 2), c4 = magc(own, 3);
    const float c0 = has_l ? halo_l<IN>(hl) : c1;
    const float c5 = has_r ? halo_r<IN>(hr) : c4;
    return chroma_taps<LEFT>(c0, c1, c2, c3, c4, c5, coff);
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

// R', G', B' of one luma row of 8 pixels in the pair layout: chroma
// 3*near + far (16x scale minus the offset, exact), Y' = (code - y_off/16) *
// 16 y_scale (one rounding: yoff = 2^23 + y_off/16, ys16 = 16 y_scale), one
// FMA per channel.
template <typename IN>
__device__ __forceinline__ void rgb_row(const F2TColour &col, float yoff, float ys16, typename Luma<IN>::V lraw,
                                        const HRow &nu, const HRow &fu, const HRow &nv, const HRow &fv,
                                        float2 (&dy)[4], float2 (&du)[4], float2 (&dv)[4], float2 (&R)[4],
                                        float2 (&G)[4], float2 (&B)[4])
{
    const float2 k3 = f2(3.0f, 3.0f);
    du[0] = ffma2(k3, nu.A, fu.A);
    du[1] = ffma2(k3, nu.B, fu.B);
    du[2] = ffma2(k3, nu.C, fu.C);
    du[3] = ffma2(k3, nu.D, fu.D);
    dv[0] = ffma2(k3, nv.A, fv.A);
    dv[1] = ffma2(k3, nv.B, fv.B);
    dv[2] = ffma2(k3, nv.C, fv.C);
    dv[3] = ffma2(k3, nv.D, fv.D);
    const float2 yo2 = f2(-yoff, -yoff), ys2 = f2(ys16, ys16);
    float2 Y[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        dy[p] = fadd2(f2(Luma<IN>::get(lraw, kP0[p]), Luma<IN>::get(lraw, kP1[p])), yo2);
        Y[p] = fmul2(dy[p], ys2);
    }
    const float2 rv2 = f2(col.r_v, col.r_v), bu2 = f2(col.b_u, col.b_u);
    const float2 gu2 = f2(-col.g_u, -col.g_u), gv2 = f2(-col.g_v, -col.g_v);
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        R[p] = ffma2(rv2, dv[p], Y[p]);
        B[p] = ffma2(bu2, du[p], Y[p]);
        G[p] = ffma2(gv2, dv[p], ffma2(gu2, du[p], Y[p]));
    }
}

// pixels (0,1) = (A.x, B.x), (2,3) = (B.y, C.x), (4,5) = (C.y, D.x), (6,7) = (D.y, A.y)
__device__ __forceinline__ void pack_row(const float2 (&R)[4], const float2 (&G)[4], const float2 (&B)[4],
                                         Row8<__half> (&o)[3])
{
    const float2(*ch[3])[4] = {&R, &G, &B};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float2(&v)[4] = *ch[c];
        o[c].v = make_uint4(pack_half2(v[0].x, v[1].x), pack_half2(v[1].y, v[2].x), pack_half2(v[2].y, v[3].x),
                            pack_half2(v[3].y, v[0].y));
    }
}
__device__ __forceinline__ void pack_row(const float2 (&R)[4], const float2 (&G)[4], const float2 (&B)[4],
                                         Row8<float> (&o)[3])
{
    const float2(*ch[3])[4] = {&R, &G, &B};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float2(&v)[4] = *ch[c];
        o[c].a = make_float4(v[0].x, v[1].x, v[1].y, v[2].x);
        o[c].b = make_float4(v[2].y, v[3].x, v[3].y, v[0].y);
    }
}

// register barriers: the rare branch below recomputes from these copies
// instead of the compiler keeping every row's intermediates live across it
__device__ __forceinline__ void opaque(HRow &h)
{
    asm volatile("" : "+f"(h.A.x), "+f"(h.A.y), "+f"(h.B.x), "+f"(h.B.y), "+f"(h.C.x), "+f"(h.C.y), "+f"(h.D.x),
                 "+f"(h.D.y));
}
__device__ __forceinline__ void opaque(uint4 &v) { asm volatile("" : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w)); }
__device__ __forceinline__ void opaque(uint2 &v) { asm volatile("" : "+r"(v.x), "+r"(v.y)); }

// The row again with its fp16 near-zero values recomputed in fp64 (rare:
// some value of the 8 pixels below 2^-11).
template <typename IN>
__device__ __forceinline__ void convert_row_tiny(const F2TColour &col, float yoff, float ys16, typename Luma<IN>::V lraw,
                                                 HRow nu, HRow fu, HRow nv, HRow fv, Row8<__half> (&o)[3])
{
    opaque(lraw);
    opaque(nu);
    opaque(fu);
    opaque(nv);
    opaque(fv);
    float2 dy[4], du[4], dv[4], R[4], G[4], B[4];
    rgb_row<IN>(col, yoff, ys16, lraw, nu, fu, nv, fv, dy, du, dv, R, G, B);
    fix_tiny_row(col, dy, du, dv, R, G, B);
    pack_row(R, G, B, o);
}

// One luma row of 8 pixels converted and packed; fp16 near-zero values
// recomputed in fp64 (rare branch).
template <typename IN, typename OUT>
__device__ __forceinline__ void convert_row(const F2TColour &col, float yoff, float ys16, typename Luma<IN>::V lraw,
                                            const HRow &nu, const HRow &fu, const HRow &nv, const HRow &fv,
                                            Row8<OUT> (&o)[3])
{
    float2 dy[4], du[4], dv[4], R[4], G[4], B[4];
    rgb_row<IN>(col, yoff, ys16, lraw, nu, fu, nv, fv, dy, du, dv, R, G, B);
    pack_row(R, G, B, o);
    if constexpr (sizeof(OUT) == 2) {
        float mn = 1.0f;
#pragma unroll
        for (int p = 0; p < 4; ++p)
            mn = fminf(mn, fminf(fminf(fminf(fabsf(R[p].x), fabsf(R[p].y)), fminf(fabsf(G[p].x), fabsf(G[p].y))),
                                 fminf(fabsf(B[p].x), fabsf(B[p].y))));
        if (mn < kF16Tiny) convert_row_tiny<IN>(col, yoff, ys16, lraw, nu, fu, nv, fv, o);
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

// p + off for a 32-bit unsigned offset: one IMAD.WIDE.U32 instead of an
// IADD3 / IADD3.X pair
__device__ __forceinline__ char *addw(char *p, uint32_t off)
{
    char *r;
    asm("mad.wide.u32 %0, %1, 1, %2;" : "=l"(r) : "r"(off), "l"(p));
    return r;
}

// Destination rows of one tile, walked row by row: ND = 1 or 2 slots held as
// pointers (one add per row and slot), ND = 0 any number (through dl).  The
// launch guarantees 2 x plane bytes < 2^32 (f2t_strip_ok).
template <typename OUT, int ND> struct DstRows {
    char *q[ND];
    uint32_t plane_b, row_b;
#ifdef NNVISR_CHECKED
    const char *lo[ND];  // checked builds: every store lands inside its (run, slot)
    int64_t slot_b;
#endif
    __device__ __forceinline__ void init(const F2TArgs &a, const DstList &dl, int x, int y)
    {
        plane_b = static_cast<uint32_t>(static_cast<int64_t>(a.Hp) * a.Wp * sizeof(OUT));
        row_b = static_cast<uint32_t>(a.Wp * sizeof(OUT));
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
            char *const qc[3] = {q[d], addw(q[d], plane_b), addw(q[d], 2 * plane_b)};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
#ifdef NNVISR_CHECKED
                NNVISR_CHECK(!pred || (qc[c] >= lo[d] && qc[c] + kPx * sizeof(OUT) <= lo[d] + slot_b));
#endif
                stg_row_if(reinterpret_cast<OUT *>(qc[c]), o[c], pred);
            }
            q[d] = addw(q[d], row_b);
        }
    }
    __device__ __forceinline__ void skip()
    {
#pragma unroll
        for (int d = 0; d < ND; ++d) q[d] = addw(q[d], row_b);
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

// Chroma row j of this thread read directly, halos included (band
// prologue, padding rows).
template <typename IN, bool LEFT>
__device__ __forceinline__ HRow chroma_row_direct(const char *ub, int64_t pitch, int j, bool live, bool has_l,
                                                  bool has_r, float coff)
{
    using V4 = typename Pack<IN>::V4;
    const IN *u = reinterpret_cast<const IN *>(ub + j * pitch);
    const V4 r = live ? *reinterpret_cast<const V4 *>(u) : V4{};
    const uint32_t sh = sizeof(IN) == 2 ? 16 : 24;
    const uint32_t hl = (has_l && live) ? static_cast<uint32_t>(load1(u - 1)) << sh : 0u;
    const uint32_t hr = (has_r && live) ? static_cast<uint32_t>(load1(u + 4)) : 0u;
    return chroma_row<IN, LEFT>(r, hl, hr, has_l, has_r, coff);
}

// Rows [y0, y1) of a band for the 8 columns at x of every thread of the CTA
// (a strip of 8 x blockDim.x columns).  Ring entry r (r = 0 .. steps) holds
// chroma row y0/2 - 1 + r (clamped to the plane) and luma rows y0 + 2r - 3
// (r >= 2) and y0 + 2r - 2 (1 <= r < steps); step s = 0 .. steps-1 emits
// luma rows y0 + 2s - 1 (s >= 1) and y0 + 2s (< the band's last real row)
// from entries s and s + 1; padding rows (y >= H) replicate row H-1.  Lanes
// whose columns are not all inside the frame run along on dummy data (their
// samples are their neighbours' halos) and are converted by the scalar path
// afterwards; lanes past the padded width store nothing.
template <typename IN, typename OUT, bool LEFT, class Dst>
__device__ __forceinline__ void march(const F2TArgs &a, const DevFrame &f, int x, int y0, int y1, Dst &dst,
                                      uint8_t *smem)
{
    using V4 = typename Pack<IN>::V4;
    using LV = typename Luma<IN>::V;
    using S = Stage<IN>;
    const int t = threadIdx.x, lane = t & 31;
    const int cw = a.W >> 1, ch = a.H >> 1, i0 = x >> 1;
    // rd: loads inside the rows (x < W; padding columns read nothing);
    // live: a tensor column (stores)
#ifdef NNVISR_STRIP_NOSTORE  // decomposition experiments only (tools/ab_decomp.sh): stores off (a.debug is 0)
    const bool rd = x < a.W, live = x < a.Wp && a.debug == 0x5eed;
#else
    const bool rd = x < a.W, live = x < a.Wp;
#endif
    const bool has_l = i0 > 0, has_r = i0 + 4 < cw;
    const float coff = kMagic + static_cast<float>(a.col.c_off >> 4);
    const float yoff = kMagic + static_cast<float>(a.col.y_off >> 4), ys16 = 16.0f * a.col.y_scale;
    const int64_t lp = f.pitch[0], up = f.pitch[1], vp = f.pitch[2];
    const char *lbase = static_cast<const char *>(f.plane[0]) + x * sizeof(IN);
    const char *ub = static_cast<const char *>(f.plane[1]) + i0 * sizeof(IN);
    const char *vb = static_cast<const char *>(f.plane[2]) + i0 * sizeof(IN);
    const uint32_t sbase = smem_addr(smem);
    const int ol = t * S::LB, oc = S::own_c(t);  // this thread's luma / chroma bytes in a stage
    const int yr1 = min(y1, a.H);
    const int steps = yr1 > y0 ? (yr1 - y0) / 2 + 1 : 0;
    if (steps > 0) {
        // running sources of the next entry to issue: luma rows y0 + 2r - 3 /
        // y0 + 2r - 2 (not read while out of the band), chroma row jn
        // clamped (advanced only inside [0, ch-1])
        const char *la = lbase + static_cast<int64_t>(y0 - 3) * lp;
        const char *lb = lbase + static_cast<int64_t>(y0 - 2) * lp;
        int jn = y0 / 2 - 1;
        const char *un = ub + static_cast<int64_t>(max(jn, 0)) * up, *vn = vb + static_cast<int64_t>(max(jn, 0)) * vp;
        // the warp's outer halo words: lane 0 the word ending at sample i0-1,
        // lane 31 the word starting at i0+4 (into the block's pads)
        const bool hv = rd && ((lane == 0 && has_l) || (lane == 31 && has_r));
        const int hsrc = lane == 0 ? -4 : S::CB, hdst = oc + hsrc;
        int ri = 0;        // next ring entry to issue
        uint32_t wofs = 0;  // its stage offset, (ri % kStages) * kBytes
        uint32_t rofs = 0;  // stage offset of the next entry to read
        auto issue = [&]() {
            const uint32_t st = sbase + wofs;
#ifdef NNVISR_STRIP_NOLOAD  // decomposition experiments only (tools/ab_decomp.sh): copies off (a.debug is 0)
            const bool in = rd && ri <= steps && a.debug == 0x5eed;
#else
            const bool in = rd && ri <= steps;
#endif
#ifdef NNVISR_CHECKED
            {  // every copy lands in its stage and reads inside its plane
                NNVISR_CHECK(static_cast<int>(blockDim.x) <= kStripThreads && ol + S::LB <= S::kL1 && S::kV + oc + S::CB <= S::kBytes &&
                             S::kU + hdst >= S::kU && S::kV + hdst + 4 <= S::kBytes);
                auto inside = [&](const char *p, int n, int pl, int rows) {
                    const char *b = static_cast<const char *>(f.plane[pl]);
                    return p >= b && p + n <= b + rows * f.pitch[pl];
                };
                NNVISR_CHECK(!(in && ri >= 2) || inside(la, S::LB, 0, a.H));
                NNVISR_CHECK(!(in && ri >= 1 && ri < steps) || inside(lb, S::LB, 0, a.H));
                NNVISR_CHECK(!in || (inside(un, S::CB, 1, ch) && inside(vn, S::CB, 2, ch)));
                NNVISR_CHECK(!(in && hv) || (inside(un + hsrc, 4, 1, ch) && inside(vn + hsrc, 4, 2, ch)));
            }
#endif
            cp_async<S::LB>(st + S::kL0 + ol, la, in && ri >= 2);
            cp_async<S::LB>(st + S::kL1 + ol, lb, in && ri >= 1 && ri < steps);
            cp_async<S::CB>(st + S::kU + oc, un, in);
            cp_async<S::CB>(st + S::kV + oc, vn, in);
            cp_async_if<4>(st + S::kU + hdst, un + hsrc, in && hv);
            cp_async_if<4>(st + S::kV + hdst, vn + hsrc, in && hv);
            cp_commit();
            la += 2 * lp;
            lb += 2 * lp;
            if (static_cast<unsigned>(jn) < static_cast<unsigned>(ch - 1)) {
                un += up;
                vn += vp;
            }
            ++jn;
            ++ri;
            wofs = wofs + S::kBytes == kStages * S::kBytes ? 0 : wofs + S::kBytes;
        };
#pragma unroll
        for (int k = 0; k < kStages - 1; ++k) issue();
        // chroma rows of entry r: own samples and the neighbours' words
        // (visible to this lane after the wait and the warp barrier)
        auto chroma_entry = [&](HRow &wu, HRow &wv) {
            const uint8_t *st = smem + rofs;
            rofs = rofs + S::kBytes == kStages * S::kBytes ? 0 : rofs + S::kBytes;
            const uint8_t *cu = st + S::kU + oc, *cv = st + S::kV + oc;
            wu = chroma_row<IN, LEFT>(*reinterpret_cast<const V4 *>(cu), *reinterpret_cast<const uint32_t *>(cu - 4),
                                      *reinterpret_cast<const uint32_t *>(cu + S::CB), has_l, has_r, coff);
            wv = chroma_row<IN, LEFT>(*reinterpret_cast<const V4 *>(cv), *reinterpret_cast<const uint32_t *>(cv - 4),
                                      *reinterpret_cast<const uint32_t *>(cv + S::CB), has_l, has_r, coff);
            return st;
        };
        // Entry r is read at step r - 1 (entry 0 before the first step).  Each
        // step waits for its entry (this lane's copies), then one warp
        // barrier makes every lane's copies of it visible AND orders the
        // neighbours' reads of the previous step before this step's issue,
        // which reuses the stage of the entry read one step ago.
        HRow bu, bv;
        cp_wait<kStages - 2>();
        __syncwarp();
        issue();
        chroma_entry(bu, bv);
        HRow cu, cv;
        // step s: chroma row y0/2 + s arrives in (wu, wv); rows y0 + 2s - 1
        // (near = previous row p, far = w; not at s = 0) and y0 + 2s (near w,
        // far p; not at the last step)
        auto step = [&](int s, HRow &pu, HRow &pv, HRow &wu, HRow &wv, bool first_row, bool second_row) {
            cp_wait<kStages - 2>();
            __syncwarp();
            issue();
            const uint8_t *st = chroma_entry(wu, wv);  // entry s + 1
            Row8<OUT> o[3];
            if (first_row) {
                convert_row<IN, OUT>(a.col, yoff, ys16, *reinterpret_cast<const LV *>(st + S::kL0 + ol), pu, wu, pv,
                                     wv, o);
                dst.put(o, live);
            }
            if (second_row) {
                convert_row<IN, OUT>(a.col, yoff, ys16, *reinterpret_cast<const LV *>(st + S::kL1 + ol), wu, pu, wv,
                                     pv, o);
                dst.put(o, live);
            }
        };
        // even steps hold (p, w) = (b, c), odd ones (c, b)
        for (int s = 0; s < steps; s += 2) {
            step(s, bu, bv, cu, cv, s >= 1, s + 1 < steps);
            if (s + 1 >= steps) break;
            step(s + 1, cu, cv, bu, bv, true, s + 2 < steps);
        }
        cp_wait<0>();  // (the tile loop's barrier orders the reads before the next tile's copies)
    }
    // padding rows (y >= H, reading A6): row H-1 (near = far = chroma row ch-1)
    if (y1 > a.H) {
        const HRow pu = chroma_row_direct<IN, LEFT>(ub, up, ch - 1, rd, has_l, has_r, coff);
        const HRow pv = chroma_row_direct<IN, LEFT>(vb, vp, ch - 1, rd, has_l, has_r, coff);
        // every lane converts (lanes outside the frame convert zeros; ragged
        // ones are redone by the scalar path), live lanes store
        const LV l = rd ? *reinterpret_cast<const LV *>(lbase + static_cast<int64_t>(a.H - 1) * lp) : LV{};
        Row8<OUT> o[3];
        convert_row<IN, OUT>(a.col, yoff, ys16, l, pu, pu, pv, pv, o);
        for (int y = max(y0, a.H); y < y1; ++y) dst.put(o, live);
    }
}

// Tile = (job, band of a.band luma rows, strip of 8 x blockDim.x columns).
// Every thread of a CTA walks the same tiles (warp-uniform loops: the march
// shuffles chroma halos between lanes).
template <typename IN, typename OUT, bool LEFT>
__global__ void __launch_bounds__(kStripThreads, NNVISR_STRIP_MINB) f2t_strip420(const F2TArgs a)
{
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int64_t tile_slot[2];
    const int bands = (a.Hp + a.band - 1) / a.band;
    const int64_t per_job = static_cast<int64_t>(bands) * a.nseg;
    // persistent CTAs, dynamic tiles: each CTA takes the launch's next tile
    // from the zeroed per-launch counter, so fast SMs take more tiles and no
    // SM idles through a long static share (r02 ncu: SMs active 86% of the
    // kernel with static striding).  The next tile's index is fetched when a
    // tile starts and published when it ends, so the atomic's latency hides
    // behind the tile (one barrier per tile, double-buffered slot).
    auto fetch = [&](int64_t i) -> int64_t {  // (no counter: static tiles b, b + G, ...)
        return a.tile_counter ? static_cast<int64_t>(atomicAdd(a.tile_counter, 1ull)) : blockIdx.x + i * gridDim.x;
    };
    if (threadIdx.x == 0) tile_slot[0] = fetch(0);
    __syncthreads();
    for (int64_t iter = 0;; ++iter) {
        const int64_t t = tile_slot[iter & 1];
        if (t >= a.tiles) break;
        int64_t nxt = 0;
        if (threadIdx.x == 0) nxt = fetch(iter + 1);
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
        if (threadIdx.x == 0) tile_slot[(iter + 1) & 1] = nxt;
        __syncthreads();  // also orders this tile's ring reads before the next tile's copies
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
    const int smem = kStages * Stage<IN>::kBytes;
    cudaError_t err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    if (err != cudaSuccess) return err;
    const int64_t slots = static_cast<int64_t>(sms) * std::max(per_sm, 1);
    // bands: ~NNVISR_F2T_STRIP_TPC (default 20) tiles per resident CTA, so
    // the dynamic schedule's tail is short, and at least 32 rows (each tile
    // start waits one memory latency before its ring fills)
    const char *e = std::getenv("NNVISR_F2T_STRIP_ROWS");
    const char *tpc_e = std::getenv("NNVISR_F2T_STRIP_TPC");
    const int64_t tpc = tpc_e && *tpc_e ? std::max(1, std::atoi(tpc_e)) : 20;
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

// The strip kernel addresses a slot's channel planes with 32-bit offsets.
bool f2t_strip_ok(int dtype, const F2TArgs &a)
{
    const int64_t plane = static_cast<int64_t>(a.Hp) * a.Wp * (dtype == kF16 ? 2 : 4);
    return 2 * plane < (static_cast<int64_t>(1) << 32);
}

// 4:2:0 RGB tensors with 16-byte aligned planes, pitches and tensor rows
// (the caller checked a.tma_ok).
cudaError_t launch_f2t_strip(int bits, int dtype, const F2TArgs &a, cudaStream_t s)
{
    if (bits == 8) return dtype == kF16 ? launch_sited<uint8_t, __half>(a, s) : launch_sited<uint8_t, float>(a, s);
    return dtype == kF16 ? launch_sited<uint16_t, __half>(a, s) : launch_sited<uint16_t, float>(a, s);
}

}  // namespace nnvisr
