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

// Tile = (job, band of a.band luma rows, strip of 8 x blockDim.x columns).
template <typename IN, typename OUT>
__global__ void __launch_bounds__(kStripThreads, 2) f2t_strip420(const F2TArgs a)
{
    using V8 = typename Pack<IN>::V8;
    const int cw = a.W >> 1, ch = a.H >> 1;
    const bool left = a.left;
    const float coff = kMagic + static_cast<float>(a.col.c_off >> 4);
    const int bands = (a.Hp + a.band - 1) / a.band;
    const int64_t per_job = static_cast<int64_t>(bands) * a.nseg;
    for (int64_t t = blockIdx.x; t < a.tiles; t += gridDim.x) {
        const int job = static_cast<int>(t / per_job);
        const int rem = static_cast<int>(t - job * per_job);
        const int band = rem / a.nseg, strip = rem - band * a.nseg;
        const int x = (strip * blockDim.x + threadIdx.x) * kPx;
        if (x >= a.Wp) continue;
        const DevFrame f = load_frame(a.frames + a.job_frame[job]);
        DstList dl;
        dl.load(a, job);
        const int y0 = band * a.band, y1 = min(y0 + a.band, a.Hp), yr1 = min(y1, a.H);
        if (x + kPx <= a.W) {
            const int i0 = x >> 1;
            const IN *lp = row_ptr<IN>(f, 0, 0) + x;
            const int64_t lpitch = f.pitch[0] / static_cast<int64_t>(sizeof(IN));
            const IN *up = row_ptr<IN>(f, 1, 0), *vp = row_ptr<IN>(f, 2, 0);
            const int64_t cpu_ = f.pitch[1] / static_cast<int64_t>(sizeof(IN)),
                          cpv = f.pitch[2] / static_cast<int64_t>(sizeof(IN));
            auto ldc = [&](int j, ChromaRaw<IN> &u, ChromaRaw<IN> &v) {
                const int jc = min(max(j, 0), ch - 1);
                u = load_chroma<IN>(up + jc * cpu_, i0, cw);
                v = load_chroma<IN>(vp + jc * cpv, i0, cw);
            };
            // march down the band's real rows [y0, yr1): step k holds chroma
            // rows b = k and c = k+1 (clamped) and emits luma row 2k+1
            // (near k, far k+1) and row 2k+2 (near k+1, far k), so every
            // chroma row is loaded and converted once (reading A5)
            if (yr1 > y0) {
                const int k0 = (y0 >> 1) - 1, k1 = (yr1 >> 1) - 1;  // steps [k0, k1]
                float bu[6], bv[6], cu[6], cvv[6];
                ChromaRaw<IN> ru, rv;
                ldc(k0, ru, rv);
                chroma_floats<IN>(ru, coff, bu);
                chroma_floats<IN>(rv, coff, bv);
                ldc(k0 + 1, ru, rv);
                V8 l0 = *reinterpret_cast<const V8 *>(lp + static_cast<int64_t>(y0) * lpitch), l1 = l0;
                for (int k = k0; k <= k1; ++k) {
                    chroma_floats<IN>(ru, coff, cu);
                    chroma_floats<IN>(rv, coff, cvv);
                    const V8 m0 = l0;  // row 2k+1 (k > k0), else row 2k+2 = y0
                    const V8 m1 = l1;  // row 2k+2 (k > k0)
                    if (k < k1) {  // issue step k+1's loads before converting step k
                        l0 = *reinterpret_cast<const V8 *>(lp + static_cast<int64_t>(2 * k + 3) * lpitch);
                        if (k + 1 < k1) l1 = *reinterpret_cast<const V8 *>(lp + static_cast<int64_t>(2 * k + 4) * lpitch);
                        ldc(k + 2, ru, rv);
                    }
                    Row8<OUT> o[3];
                    if (k > k0) {  // row 2k+1: near k (b), far k+1 (c)
                        convert_row<IN, OUT>(a.col, left, m0, bu, cu, bv, cvv, o);
                        store_row<OUT>(a, dl, o, x, 2 * k + 1);
                    }
                    if (k < k1) {  // row 2k+2: near k+1 (c), far k (b)
                        convert_row<IN, OUT>(a.col, left, k > k0 ? m1 : m0, cu, bu, cvv, bv, o);
                        store_row<OUT>(a, dl, o, x, 2 * k + 2);
                    }
#pragma unroll
                    for (int t = 0; t < 6; ++t) {
                        bu[t] = cu[t];
                        bv[t] = cvv[t];
                    }
                }
            }
            // padding rows (y >= H, reading A6): row H-1 (near = far = chroma row ch-1)
            if (y1 > a.H && max(y0, a.H) < y1) {
                float pu[6], pv[6];
                ChromaRaw<IN> ru, rv;
                ldc(ch - 1, ru, rv);
                chroma_floats<IN>(ru, coff, pu);
                chroma_floats<IN>(rv, coff, pv);
                const V8 l = *reinterpret_cast<const V8 *>(lp + static_cast<int64_t>(a.H - 1) * lpitch);
                Row8<OUT> o[3];
                convert_row<IN, OUT>(a.col, left, l, pu, pu, pv, pv, o);
                for (int y = max(y0, a.H); y < y1; ++y) store_row<OUT>(a, dl, o, x, y);
            }
        } else {
            for (int y = y0; y < y1; ++y) slow_row<IN, OUT>(a, dl, f, x, y);
        }
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
    int per_sm = 0;
    cudaError_t err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0);
    if (err != cudaSuccess) return err;
    const int64_t grid = std::min<int64_t>(a.tiles, static_cast<int64_t>(sms) * std::max(per_sm, 1) * 4);
    kernel<<<static_cast<int>(grid), threads, 0, s>>>(a);
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
