// kernels_strip.cu -- frames -> tensor for LOW FAN-OUT launches of 4:2:0
// clips: store mode S (each clip frame
// converted once into a frame-major store, §3.3 P:373-382 at batch
// 1), the Fig. 1 batch slots (NEXT-2) and 2-frame windows (c4), where every
// converted frame is written to at most two tensor slots.
//
// There the conversion itself, not HBM, bounds the TMA pipeline of
// kernels_tma.cu (profiles/r01: issue active 56% at 4.0 TB/s in c2 store
// mode, ~35 instructions per pixel, a third of them barrier waits, per-pixel
// branches and address arithmetic).  This kernel is the lean form of the same
// arithmetic:
//
//   * a thread owns 8 luma columns and MARCHES DOWN a band of rows, so each
//     4:2:0 chroma row is loaded and converted once per band (not three times
//     per row pair): luma row 2j takes 3 x chroma row j + row j-1, row 2j+1
//     3 x row j + row j+1 (reading A5, clamped), and rows j-1, j, j+1 rotate
//     through registers;
//   * loads are plain 128-bit LDGs straight from the frame (the next row
//     pair's loads are issued before the current pair is converted), stores
//     are 128-bit STGs straight into every destination slot: no shared
//     memory, no barriers, no producer/consumer hand-offs;
//   * the fp16 near-zero test (f2t_fix_tiny) is one vote per 8 pixels, the
//     fp64 recompute only inside that rare branch.
//
// The arithmetic is the TMA fast path's operation for operation (magic-number
// integer->float, exact integer chroma sums, one rounding of Y', one FMA per
// channel), so both kernels give bit-identical tensors (tests compare them).
#include <algorithm>

#include "common.cuh"

namespace nnvisr {
namespace {
using namespace dev;

constexpr int kStripThreads = 256;

// 4 chroma samples at i0 (vector) and the two neighbours i0-1, i0+4
// (clamped to the plane): raw codes.
template <typename IN> struct ChromaRaw {
    typename Pack<IN>::V4 v;
    int l, r;
};

template <typename IN>
__device__ __forceinline__ ChromaRaw<IN> load_chroma(const IN *row, int i0, int cw)
{
    ChromaRaw<IN> c;
    c.v = *reinterpret_cast<const typename Pack<IN>::V4 *>(row + i0);
    c.l = load1(row + max(i0 - 1, 0));
    c.r = load1(row + min(i0 + 4, cw - 1));
    return c;
}

// raw codes -> floats code - c_off/16 (exact): f[0] = i0-1, f[1..4], f[5] = i0+4
template <typename IN>
__device__ __forceinline__ void chroma_floats(const ChromaRaw<IN> &c, float coff, float (&f)[6])
{
    mag4(c.v, &f[1]);
    f[0] = mag(kMagicBits | static_cast<uint32_t>(c.l));
    f[5] = mag(kMagicBits | static_cast<uint32_t>(c.r));
#pragma unroll
    for (int t = 0; t < 6; t += 2) {
        const float2 d = __fadd2_rn(make_float2(f[t], f[t + 1]), make_float2(-coff, -coff));
        f[t] = d.x;
        f[t + 1] = d.y;
    }
}

// One luma row of 8 pixels from its near / far chroma rows (both planes):
// the TMA fast path's arithmetic (kernels_tma.cu f2t_tma, 4:2:0 branch).
// fp16 outputs are packed pixel pair by pair (few live registers); if any of
// the 24 values is below 2^-11 the row is redone with the per-pixel fp64
// recompute (f2t_fix_tiny), a rare branch.
template <typename IN>
__device__ __forceinline__ void chroma_h(bool left, const float (&n)[6], const float (&f)[6], float (&cd)[kPx])
{
    float v[6];
#pragma unroll
    for (int t = 0; t < 6; t += 2) {
        const float2 v2 = __ffma2_rn(make_float2(3.0f, 3.0f), make_float2(n[t], n[t + 1]), make_float2(f[t], f[t + 1]));
        v[t] = v2.x;
        v[t + 1] = v2.y;
    }
    if (!left) {
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const float2 h2 = __ffma2_rn(make_float2(3.0f, 3.0f), make_float2(v[m + 1], v[m + 1]),
                                         make_float2(v[m], v[m + 2]));
            cd[2 * m] = h2.x;
            cd[2 * m + 1] = h2.y;
        }
    } else {  // LEFT (MPEG-2): co-sited even columns, (1/2, 1/2) odd
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            cd[2 * m] = 4.0f * v[m + 1];
            cd[2 * m + 1] = 2.0f * (v[m + 1] + v[m + 2]);
        }
    }
}

template <typename IN, typename OUT>
__device__ __forceinline__ void convert_row(const F2TColour &col, bool left, typename Pack<IN>::V8 lraw,
                                            const float (&nu)[6], const float (&fu)[6], const float (&nv)[6],
                                            const float (&fv)[6], Row8<OUT> (&o)[3])
{
    float du[kPx], dv[kPx];
    chroma_h<IN>(left, nu, fu, du);
    chroma_h<IN>(left, nv, fv, dv);
    float dy[kPx];
    mag8(lraw, dy);
    const float yoff = kMagic + static_cast<float>(col.y_off >> 4);
    const float ys16 = 16.0f * col.y_scale;
    const float2 yo2 = make_float2(-yoff, -yoff), ys2 = make_float2(ys16, ys16);
    const float2 rv2 = make_float2(col.r_v, col.r_v), bu2 = make_float2(col.b_u, col.b_u);
    const float2 gu2 = make_float2(-col.g_u, -col.g_u), gv2 = make_float2(-col.g_v, -col.g_v);
    if constexpr (sizeof(OUT) == 2) {
        uint32_t pr[4], pg[4], pb[4];
        float mn = 1.0f;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const float2 d = __fadd2_rn(make_float2(dy[2 * m], dy[2 * m + 1]), yo2);
            const float2 Y = __fmul2_rn(d, ys2);
            const float2 u2 = make_float2(du[2 * m], du[2 * m + 1]), v2 = make_float2(dv[2 * m], dv[2 * m + 1]);
            const float2 R2 = __ffma2_rn(rv2, v2, Y), B2 = __ffma2_rn(bu2, u2, Y);
            const float2 G2 = __ffma2_rn(gv2, v2, __ffma2_rn(gu2, u2, Y));
            mn = fminf(mn, fminf(fminf(fabsf(R2.x), fabsf(R2.y)), fminf(fminf(fabsf(G2.x), fabsf(G2.y)),
                                                                       fminf(fabsf(B2.x), fabsf(B2.y)))));
            pr[m] = pack_half2(R2.x, R2.y);
            pg[m] = pack_half2(G2.x, G2.y);
            pb[m] = pack_half2(B2.x, B2.y);
        }
        if (mn < kF16Tiny) {  // rare: redo the row with the fp64 near-zero recompute
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                float R[2], G[2], B[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int k = 2 * m + e;
                    const float d = dy[k] - yoff, Y = d * ys16;
                    R[e] = fmaf(col.r_v, dv[k], Y);
                    B[e] = fmaf(col.b_u, du[k], Y);
                    G[e] = fmaf(-col.g_v, dv[k], fmaf(-col.g_u, du[k], Y));
                    f2t_fix_tiny<OUT>(col, d, du[k], dv[k], R[e], G[e], B[e]);
                }
                pr[m] = pack_half2(R[0], R[1]);
                pg[m] = pack_half2(G[0], G[1]);
                pb[m] = pack_half2(B[0], B[1]);
            }
        }
        o[0].v = make_uint4(pr[0], pr[1], pr[2], pr[3]);
        o[1].v = make_uint4(pg[0], pg[1], pg[2], pg[3]);
        o[2].v = make_uint4(pb[0], pb[1], pb[2], pb[3]);
    } else {
        float R[kPx], G[kPx], B[kPx];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const float2 d = __fadd2_rn(make_float2(dy[2 * m], dy[2 * m + 1]), yo2);
            const float2 Y = __fmul2_rn(d, ys2);
            const float2 u2 = make_float2(du[2 * m], du[2 * m + 1]), v2 = make_float2(dv[2 * m], dv[2 * m + 1]);
            const float2 R2 = __ffma2_rn(rv2, v2, Y), B2 = __ffma2_rn(bu2, u2, Y);
            const float2 G2 = __ffma2_rn(gv2, v2, __ffma2_rn(gu2, u2, Y));
            R[2 * m] = R2.x;
            R[2 * m + 1] = R2.y;
            G[2 * m] = G2.x;
            G[2 * m + 1] = G2.y;
            B[2 * m] = B2.x;
            B[2 * m + 1] = B2.y;
        }
        o[0].set(R);
        o[1].set(G);
        o[2].set(B);
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

// Destination rows of one tile, walked row by row: ND = 1 or 2 slots held as
// pointers (one 64-bit add per row and slot), ND = 0 any number (dl).
template <typename OUT, int ND> struct DstRows {
    OUT *q[ND];
    int64_t plane;
    int wp;
    __device__ __forceinline__ void init(const F2TArgs &a, const DstList &dl, int x, int y)
    {
        plane = static_cast<int64_t>(a.Hp) * a.Wp;
        wp = a.Wp;
#pragma unroll
        for (int d = 0; d < ND; ++d) {
            const int cd = dl.code[d];
            q[d] = reinterpret_cast<OUT *>(a.dst + static_cast<int64_t>(cd >> 5) * a.run_stride +
                                           static_cast<int64_t>(cd & 31) * a.slot_bytes) +
                   static_cast<int64_t>(y) * a.Wp + x;
        }
    }
    __device__ __forceinline__ void put(const Row8<OUT> (&o)[3])
    {
#pragma unroll
        for (int d = 0; d < ND; ++d) {
#pragma unroll
            for (int c = 0; c < 3; ++c) o[c].store(q[d] + c * plane);
            q[d] += wp;
        }
    }
    __device__ __forceinline__ void skip()
    {
#pragma unroll
        for (int d = 0; d < ND; ++d) q[d] += wp;
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
    __device__ __forceinline__ void put(const Row8<OUT> (&o)[3]) { store_row<OUT>(*a, *dl, o, x, y++); }
    __device__ __forceinline__ void skip() { ++y; }
};

// ---- per-thread asynchronous copies (cp.async, LDGSTS): the loads of the
// next kStages steps wait in shared memory instead of registers, so each
// warp keeps several steps of HBM reads in flight at 128 registers.
__device__ __forceinline__ uint32_t smem_addr(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
template <int BYTES>
__device__ __forceinline__ void cp_async(void *dst, const void *src, bool valid)
{
    const int n = valid ? BYTES : 0;  // 0: zero-fill, nothing read
    if constexpr (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src), "r"(n) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(smem_addr(dst)), "l"(src), "n"(BYTES),
                     "r"(n)
                     : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr int kStages = 4;  // steps in flight per thread

// One pipeline stage = one march step of every thread of the CTA, structure
// of arrays (conflict-free vector reads): luma rows 2k+1, 2k+2 (8 samples
// each), chroma row k+1 of both planes (4 samples each), and per warp the
// 4-byte words holding the warp's outer halo samples (lane 0: i0-1, lane 31:
// i0+4) of both planes.
template <typename IN> struct StageLayout {
    static constexpr int LB = 8 * sizeof(IN), CB = 4 * sizeof(IN);  // luma / chroma bytes per thread
    __host__ __device__ static constexpr int bytes(int threads) { return threads * (2 * LB + 2 * CB) + (threads / 32) * 16; }
    __device__ static uint8_t *l0(uint8_t *st, int t) { return st + t * LB; }
    __device__ static uint8_t *l1(uint8_t *st, int t, int n) { return st + n * LB + t * LB; }
    __device__ static uint8_t *u(uint8_t *st, int t, int n) { return st + 2 * n * LB + t * CB; }
    __device__ static uint8_t *v(uint8_t *st, int t, int n) { return st + 2 * n * LB + n * CB + t * CB; }
    __device__ static uint32_t *halo(uint8_t *st, int w, int n) { return reinterpret_cast<uint32_t *>(st + 2 * n * (LB + CB)) + 4 * w; }
};

// halo samples inside their aligned 4-byte words: left word ends at sample
// i0-1, right word starts at sample i0+4
template <typename IN> __device__ __forceinline__ uint32_t halo_left(uint32_t w)
{
    return sizeof(IN) == 2 ? (w >> 16) : (w >> 24);
}
template <typename IN> __device__ __forceinline__ uint32_t halo_right(uint32_t w)
{
    return sizeof(IN) == 2 ? (w & 0xffffu) : (w & 0xffu);
}

// Chroma row k+1 of this thread from the stage: own 4 samples, halos from the
// neighbouring lanes (shuffles) or, at warp edges, from the halo words;
// clamped at the plane edges (reading A5).  Every lane of the warp calls it.
template <typename IN>
__device__ __forceinline__ void stage_chroma(const uint8_t *own, uint32_t hl, uint32_t hr, int lane, bool has_l,
                                             bool has_r, float coff, float (&f)[6])
{
    mag4(*reinterpret_cast<const typename Pack<IN>::V4 *>(own), &f[1]);
    const float up = __shfl_up_sync(0xffffffffu, f[4], 1), dn = __shfl_down_sync(0xffffffffu, f[1], 1);
    f[0] = !has_l ? f[1] : lane == 0 ? mag(kMagicBits | halo_left<IN>(hl)) : up;
    f[5] = !has_r ? f[4] : lane == 31 ? mag(kMagicBits | halo_right<IN>(hr)) : dn;
#pragma unroll
    for (int t = 0; t < 6; t += 2) {
        const float2 d = __fadd2_rn(make_float2(f[t], f[t + 1]), make_float2(-coff, -coff));
        f[t] = d.x;
        f[t + 1] = d.y;
    }
}

// The rows [y0, y1) of a band for the 8 columns at x of every thread (one
// CTA = a strip of 8 x blockDim.x columns).  Real rows are marched step by
// step with cp.async prefetch kStages steps ahead; padding rows (y >= H)
// replicate row H-1.  Lanes whose columns are not all inside the frame
// (x + 8 > W) run along with dummy data and are converted afterwards by the
// scalar path; lanes past the padded width store nothing.
template <typename IN, typename OUT, class Dst>
__device__ __forceinline__ void march(const F2TArgs &a, const DevFrame &f, int x, int y0, int y1, Dst &dst,
                                      uint8_t *smem)
{
    using V8 = typename Pack<IN>::V8;
    using SL = StageLayout<IN>;
    const int n = blockDim.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int cw = a.W >> 1, ch = a.H >> 1, i0 = x >> 1;
    const bool fast = x + kPx <= a.W, live = x < a.Wp;
    const bool has_l = i0 > 0, has_r = i0 + 4 < cw;
    const bool left = a.left;
    const float coff = kMagic + static_cast<float>(a.col.c_off >> 4);
    const int64_t lp = f.pitch[0], up = f.pitch[1], vp = f.pitch[2];
    const char *lbase = static_cast<const char *>(f.plane[0]) + x * sizeof(IN);
    const char *ub = static_cast<const char *>(f.plane[1]) + i0 * sizeof(IN);
    const char *vb = static_cast<const char *>(f.plane[2]) + i0 * sizeof(IN);
    const int stage_bytes = (SL::bytes(n) + 15) / 16 * 16;
    const int yr1 = min(y1, a.H);
    // step s: luma rows y0 + 2s - 1 (s >= 1) and y0 + 2s (< yr1), chroma row y0/2 + s (clamped)
    const int steps = yr1 > y0 ? (yr1 - y0) / 2 + 1 : 0;
    auto issue = [&](int s) {
        uint8_t *st = smem + (s % kStages) * stage_bytes;
        const int ya = y0 + 2 * s - 1, yb = y0 + 2 * s;
        const bool in = live && s < steps;
        cp_async<SL::LB>(SL::l0(st, t), lbase + max(ya, 0) * lp, in && s >= 1);
        cp_async<SL::LB>(SL::l1(st, t, n), lbase + min(yb, a.H - 1) * lp, in && yb < yr1);
        const int jc = min(y0 / 2 + s, ch - 1);
        const char *u = ub + jc * up, *v = vb + jc * vp;
        cp_async<SL::CB>(SL::u(st, t, n), u, in);
        cp_async<SL::CB>(SL::v(st, t, n), v, in);
        if (lane == 0 || lane == 31) {
            uint32_t *hw = SL::halo(st, w, n) + (lane == 31 ? 2 : 0);
            const int off = lane == 0 ? -4 : 4 * static_cast<int>(sizeof(IN));  // aligned words around i0-1 / i0+4
            const bool hv = in && (lane == 0 ? has_l : has_r);
            cp_async<4>(hw, u + (hv ? off : 0), hv);
            cp_async<4>(hw + 1, v + (hv ? off : 0), hv);
        }
        cp_commit();
    };
    if (steps > 0) {
        for (int s = 0; s < kStages - 1; ++s) issue(s);
        // chroma row y0/2 - 1 (clamped): the far row of the band's first luma row
        float bu[6], bv[6], cu[6], cvv[6];
        {
            const int jb = max(y0 / 2 - 1, 0);
            const IN *u = reinterpret_cast<const IN *>(ub + jb * up), *v = reinterpret_cast<const IN *>(vb + jb * vp);
            const typename Pack<IN>::V4 zu = live ? *reinterpret_cast<const typename Pack<IN>::V4 *>(u)
                                                  : typename Pack<IN>::V4{};
            const typename Pack<IN>::V4 zv = live ? *reinterpret_cast<const typename Pack<IN>::V4 *>(v)
                                                  : typename Pack<IN>::V4{};
            const uint32_t hlu = (lane == 0 && has_l && live) ? load1(u - 1) : 0, hlv = (lane == 0 && has_l && live) ? load1(v - 1) : 0;
            const uint32_t hru = (lane == 31 && has_r && live) ? load1(u + 4) : 0, hrv = (lane == 31 && has_r && live) ? load1(v + 4) : 0;
            // (raw samples, so place them where halo_left/right expect them)
            const uint32_t sh = sizeof(IN) == 2 ? 16 : 24;
            stage_chroma<IN>(reinterpret_cast<const uint8_t *>(&zu), hlu << sh, hru, lane, has_l, has_r, coff, bu);
            stage_chroma<IN>(reinterpret_cast<const uint8_t *>(&zv), hlv << sh, hrv, lane, has_l, has_r, coff, bv);
        }
        // step s converts chroma row y0/2 + s into (wu, wv); rows
        // 2k+1 = y0 + 2s - 1 (near = previous row, far = this one) and
        // 2k+2 = y0 + 2s (near this one, far the previous)
        auto step = [&](int s, float (&pu)[6], float (&pv)[6], float (&wu)[6], float (&wv)[6]) {
            issue(s + kStages - 1);
            cp_wait<kStages - 1>();
            const uint8_t *st = smem + (s % kStages) * stage_bytes;
            const uint32_t *hw = SL::halo(const_cast<uint8_t *>(st), w, n);
            stage_chroma<IN>(SL::u(const_cast<uint8_t *>(st), t, n), hw[0], hw[2], lane, has_l, has_r, coff, wu);
            stage_chroma<IN>(SL::v(const_cast<uint8_t *>(st), t, n), hw[1], hw[3], lane, has_l, has_r, coff, wv);
            const int ya = y0 + 2 * s - 1, yb = ya + 1;
            Row8<OUT> o[3];
            if (s >= 1) {
                const V8 l = *reinterpret_cast<const V8 *>(SL::l0(const_cast<uint8_t *>(st), t));
                convert_row<IN, OUT>(a.col, left, l, pu, wu, pv, wv, o);
                if (fast) dst.put(o);
                else dst.skip();
            }
            if (yb < yr1) {
                const V8 l = *reinterpret_cast<const V8 *>(SL::l1(const_cast<uint8_t *>(st), t, n));
                convert_row<IN, OUT>(a.col, left, l, wu, pu, wv, pv, o);
                if (fast) dst.put(o);
                else dst.skip();
            }
        };
        for (int s = 0; s < steps; s += 2) {
            step(s, bu, bv, cu, cvv);
            if (s + 1 >= steps) break;
            step(s + 1, cu, cvv, bu, bv);
        }
        cp_wait<0>();
    }
    // padding rows (y >= H, reading A6): row H-1 (near = far = chroma row ch-1)
    if (y1 > a.H && fast) {
        float pu[6], pv[6];
        const IN *u = reinterpret_cast<const IN *>(ub + (ch - 1) * up), *v = reinterpret_cast<const IN *>(vb + (ch - 1) * vp);
        ChromaRaw<IN> ru = load_chroma<IN>(u - i0, i0, cw), rv = load_chroma<IN>(v - i0, i0, cw);
        chroma_floats<IN>(ru, coff, pu);
        chroma_floats<IN>(rv, coff, pv);
        const V8 l = *reinterpret_cast<const V8 *>(lbase + static_cast<int64_t>(a.H - 1) * lp);
        Row8<OUT> o[3];
        convert_row<IN, OUT>(a.col, left, l, pu, pu, pv, pv, o);
        for (int y = max(y0, a.H); y < y1; ++y) dst.put(o);
    }
}

// Tile = (job, band of a.band luma rows, strip of 8 x blockDim.x columns).
// Every thread of a CTA walks the same tiles (warp-uniform loops: the march
// shuffles chroma halos between lanes).
template <typename IN, typename OUT>
__global__ void __launch_bounds__(kStripThreads, 2) f2t_strip420(const F2TArgs a)
{
    extern __shared__ __align__(16) uint8_t smem[];
    const int bands = (a.Hp + a.band - 1) / a.band;
    const int64_t per_job = static_cast<int64_t>(bands) * a.nseg;
    for (int64_t t = blockIdx.x; t < a.tiles; t += gridDim.x) {
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
            march<IN, OUT>(a, f, x, y0, y1, d, smem);
        } else if (dl.nd == 2) {
            DstRows<OUT, 2> d;
            d.init(a, dl, x, y0);
            march<IN, OUT>(a, f, x, y0, y1, d, smem);
        } else {
            DstRows<OUT, 0> d;
            d.init(a, dl, x, y0);
            march<IN, OUT>(a, f, x, y0, y1, d, smem);
        }
        if (x < a.Wp && x + kPx > a.W) {  // ragged right edge / padding columns: scalar path
            for (int y = y0; y < y1; ++y) slow_row<IN, OUT>(a, dl, f, x, y);
        }
        __syncwarp();  // the stage ring is reused by the next tile
    }
}

template <typename IN, typename OUT>
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
    const int threads = std::min(kStripThreads, (groups + 31) / 32 * 32);
    a.nseg = (groups + threads - 1) / threads;
    const char *e = std::getenv("NNVISR_F2T_STRIP_ROWS");
    a.band = e && *e ? std::max(2, std::atoi(e) & ~1) : 32;
    const int bands = (a.Hp + a.band - 1) / a.band;
    a.tiles = a.jobs * bands * a.nseg;
    if (a.tiles <= 0) return cudaSuccess;
    auto kernel = f2t_strip420<IN, OUT>;
    const int smem = kStages * ((StageLayout<IN>::bytes(threads) + 15) / 16 * 16);
    cudaError_t err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    if (err != cudaSuccess) return err;
    const int64_t grid = std::min<int64_t>(a.tiles, static_cast<int64_t>(sms) * std::max(per_sm, 1) * 4);
    kernel<<<static_cast<int>(grid), threads, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace

// 4:2:0 RGB tensors with 16-byte aligned planes, pitches and tensor rows
// (the caller checked a.tma_ok).
cudaError_t launch_f2t_strip(int bits, int dtype, const F2TArgs &a, cudaStream_t s)
{
    if (bits == 8) return dtype == kF16 ? launch<uint8_t, __half>(a, s) : launch<uint8_t, float>(a, s);
    return dtype == kF16 ? launch<uint16_t, __half>(a, s) : launch<uint16_t, float>(a, s);
}

}  // namespace nnvisr
