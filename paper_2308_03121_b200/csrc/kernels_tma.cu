// kernels_tma.cu -- TMA-pipelined conversion kernels (sm_100a).
//
// The hot path is a pair of streaming passes (SURVEY.md §8(a) A3-A7 and
// B1-B4).  All kernels here are persistent, warp-specialised pipelines:
//
//  * a tile is a band of row units (a 4:2:0 row pair, else one row) times a
//    segment of up to 2048 columns (8 columns per consumer thread; 4:2:0
//    frames up to 4096 columns can be one "wide" whole-row segment);
//  * tiles are handed out dynamically: each launch uploads a zeroed tile
//    counter with its work tables and one thread per CTA fetches tiles in
//    order (TileSource), so fast SMs take more tiles;
//  * one thread stages each tile into a shared-memory stage with TMA bulk
//    copies (cp.async.bulk.shared::cluster.global, completion counted in bytes
//    on the stage's `full` mbarrier) and writes the stage's tile header --
//    for frames->tensor the band's luma rows with their co-sited chroma rows
//    and one-row halo (north_star: "TMA or shared-memory staging of luma tiles
//    together with their co-sited chroma rows"), for tensor->frames the
//    tile's R', G', B' (or luma and chroma) rows;
//  * consumer warps convert from shared memory while the next stages load;
//    f2t writes the converted band to an output buffer that storer threads fan
//    out to every tuple slot holding the frame with TMA bulk stores
//    (cp.async.bulk.global.shared::cta); t2f stores codes with st.global.
//
// Coordinates outside the frame are clamped when shared memory is read
// (padding replicates the last row/column, reading A6; chroma taps clamp to
// the plane, reading A5), so no copy ever leaves the plane: the copy windows
// are clamped to the plane and 16-byte aligned.  The host enables this path
// only when every window is 16-byte aligned (see nnvisr.cpp, tma_ok).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace nnvisr {
namespace {
using namespace dev;

// ---------------------------------------------------------------- TMA / mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t"
        ".reg .pred P1;\n\t"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra DONE;\n\t"
        "bra LAB_WAIT;\n\t"
        "DONE:\n\t"
        "}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680u)  // suspend-time hint: sleep until the phase completes, fewer polls
        : "memory");
}
// global -> shared bulk copy (TMA engine; SASS UBLKCP), completes on `bar`.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    NNVISR_CHECK(((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | bytes) & 15) == 0);
    NNVISR_CHECK_SMEM(dst, bytes);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// shared -> global bulk store (TMA engine), tracked by bulk groups
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes)
{
    NNVISR_CHECK(((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | bytes) & 15) == 0);
    NNVISR_CHECK_SMEM(src, bytes);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
// wait until at most n (>= 0) of this thread's bulk groups are still reading
// shared memory (n > 7: 7, i.e. waits longer than needed)
__device__ __forceinline__ void bulk_wait_read_le(int n)
{
    switch (n) {
    case 0: bulk_wait_read<0>(); break;
    case 1: bulk_wait_read<1>(); break;
    case 2: bulk_wait_read<2>(); break;
    case 3: bulk_wait_read<3>(); break;
    case 4: bulk_wait_read<4>(); break;
    case 5: bulk_wait_read<5>(); break;
    case 6: bulk_wait_read<6>(); break;
    default: bulk_wait_read<7>(); break;
    }
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Experiment timeline (build with -DNNVISR_F2T_TRACE, run with
// NNVISR_F2T_DEBUG=8): SM clock of event `ev` of tile i, CTAs 0 and 1, first
// 128 tiles (see f2t_tma_launch).  Compiled out otherwise.
constexpr int kTraceTiles = 128, kTraceEvents = 8, kTraceCtas = 1024;
#ifdef NNVISR_F2T_TRACE
__device__ __forceinline__ uint64_t gtimer()
{
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t smid()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
#endif
#ifdef NNVISR_F2T_TRACE
#define NNVISR_TRACE(cond, ev, i)                                                                 \
    do {                                                                                          \
        if ((cond) && (a.debug & 8) && blockIdx.x < 2 && (i) < kTraceTiles)                       \
            a.trace[(blockIdx.x * kTraceEvents + (ev)) * kTraceTiles + (i)] = clock64();          \
    } while (0)
// per-CTA record after the tile timelines: [start ns, end ns, smid] (globaltimer)
#define NNVISR_TRACE_CTA(slot, val)                                                                   \
    do {                                                                                              \
        if ((a.debug & 8) && blockIdx.x < kTraceCtas)                                                 \
            a.trace[2 * kTraceEvents * kTraceTiles + 3 * blockIdx.x + (slot)] = (val);               \
    } while (0)
#else
#define NNVISR_TRACE_CTA(slot, val) \
    do {                            \
    } while (0)
#define NNVISR_TRACE(cond, ev, i) \
    do {                          \
    } while (0)
#endif

constexpr int kSegW = kThreads * kPx;         // columns per tile segment (2048)
constexpr int kMaxStages = 8;
constexpr int kMaxOutBufs = 8;
// per-stage tile header written by the loader, read by the consumers
struct F2THdr {
    int u0, nu, x0, x1, ly0, cy0, lw0, cw0;
};
// mbarriers (full, empty per stage; ofree, conv per output buffer), the
// stage headers and the ring of local tile -> launch tile ids (f2t) at the
// start of dynamic smem
constexpr int kTileRing = 16;  // >= stages + output buffers + 1
constexpr int kBarBytes = 8 * (2 * kMaxStages + 2 * kMaxOutBufs) + 32 * kMaxStages + 8 * kTileRing;

// The tiles one CTA processes, in order: dynamic (a zeroed per-launch
// counter: each fetch takes the next unprocessed tile of the launch, so fast
// SMs take more tiles and no CTA is left finishing a long static share; every
// CTA ends with exactly one fetch past the end) or, without a counter,
// static (tiles b, b + G, ...).  One thread per CTA fetches, in order.
struct TileSource {
    unsigned long long *counter;
    int64_t tiles, next;
    // skip: local tiles fetched by another thread first (static mode)
    __device__ __forceinline__ void init(unsigned long long *c, int64_t n, int skip = 0)
    {
        counter = c;
        tiles = n;
        next = blockIdx.x + static_cast<int64_t>(skip) * gridDim.x;
    }
    // next tile of this CTA, or -1 when the launch has none left
    __device__ __forceinline__ int64_t fetch()
    {
        int64_t t;
        if (counter) {
            t = static_cast<int64_t>(atomicAdd(counter, 1ull));
        } else {
            t = next;
            next += gridDim.x;
        }
        return t < tiles ? t : -1;
    }
};

// tile -> (job, row unit, segment)
__device__ __forceinline__ void decode_tile(int64_t t, int rowunits, int nseg, int seg_w, int &job, int &ru, int &x0)
{
    const int64_t per_job = static_cast<int64_t>(rowunits) * nseg;
    job = static_cast<int>(t / per_job);
    const int rem = static_cast<int>(t - static_cast<int64_t>(job) * per_job);
    ru = rem / nseg;
    x0 = (rem - ru * nseg) * seg_w;
}

// ------------------------------------------------------------------ f2t
// A tile is a band of B row units (4:2:0 row pairs, else rows) of one column
// segment of one distinct frame.  Stage layout (samples of IN):
//   4:2:0     luma rows [2B][ls] | U rows [B+2][cs] | V rows [B+2][cs]
//   4:4:4/RGB plane p rows [B][ls], p = 0, 1, 2
// holding the band's rows clamped to the frame (padding rows replicate row
// H-1): luma rows ly0..ly1 and chroma rows cy0..cy1, the near and far chroma
// rows of every luma row of the band.  With a single segment whose staged row
// stride equals the plane pitch (a.whole) each plane's band rows arrive in ONE
// bulk copy; otherwise one copy per row of the segment's window.
template <int FAMILY, typename IN> struct F2TStage {
    static constexpr int G = 16 / sizeof(IN);  // samples per 16 bytes
    static constexpr int ROWS = FAMILY == kYUV420 ? 2 : 1;
    int ls, cs, B;  // luma / chroma staged row strides (samples), band height
    __device__ __host__ F2TStage(int ls_, int cs_, int B_) : ls(ls_), cs(cs_), B(B_) {}
    __device__ __host__ int bytes() const
    {
        return FAMILY == kYUV420 ? (2 * B * ls + 2 * (B + 2) * cs) * (int)sizeof(IN) : 3 * B * ls * (int)sizeof(IN);
    }
    __device__ IN *luma(uint8_t *st, int row) const { return reinterpret_cast<IN *>(st) + row * ls; }
    __device__ IN *chroma(uint8_t *st, int p, int row) const
    {
        return reinterpret_cast<IN *>(st) + 2 * B * ls + (p * (B + 2) + row) * cs;
    }
    __device__ IN *plane(uint8_t *st, int p, int row) const { return reinterpret_cast<IN *>(st) + (p * B + row) * ls; }
};

// A vector of staged samples (checked builds: inside the tile's stage).
template <typename V>
__device__ __forceinline__ V ld_stage(const void *p, const uint8_t *st, int stage_bytes)
{
    NNVISR_CHECK(static_cast<const uint8_t *>(p) >= st && static_cast<const uint8_t *>(p) + sizeof(V) <= st + stage_bytes);
    (void)st;
    (void)stage_bytes;
    return *reinterpret_cast<const V *>(p);
}

// Copy windows of a segment [x0, x1): luma [lw0, lw1), chroma [cw0, cw1).
struct F2TWindow {
    int lw0, lw1, cw0, cw1;
    __device__ __forceinline__ void set(int x0, int x1, int W, int G, bool chroma420)
    {
        // window ends are rounded up to whole 16-byte groups: a width that is
        // not a multiple of 16 bytes reads into the row's pitch padding (the
        // host requires 16-byte pitches), never past the row's allocation
        const int xr = min(x1, W);
        if (x0 < W) {
            lw0 = x0;
            lw1 = (xr + G - 1) / G * G;
        } else {  // a segment of padding columns only: they replicate column W-1
            lw0 = (W - 1) / G * G;
            lw1 = (W + G - 1) / G * G;
        }
        if (chroma420) {
            const int cw = W >> 1;
            const int lo = (min(x0, W - 1) >> 1) - 1;
            cw0 = max(0, (lo >= 0 ? lo : -G) / G * G);
            cw1 = min((cw + G - 1) / G * G, ((xr >> 1) + 1 + G - 1) / G * G);
        }
    }
};

// tile -> (job, band, segment start); band = row units [band*B, min(band*B + B, rowunits))
struct F2TTile {
    int job, u0, nu, x0, x1, ly0, ly1, cy0, cy1;
    __device__ __forceinline__ void set(const F2TArgs &a, int64_t t, int ROWS)
    {
        const int bands = (a.rowunits + a.band - 1) / a.band;
        int band;
        decode_tile(t, bands, a.nseg, a.fsegw, job, band, x0);
        x1 = min(x0 + a.fsegw, a.Wp);
        u0 = band * a.band;
        nu = min(a.band, a.rowunits - u0);
        ly0 = min(u0 * ROWS, a.H - 1);
        ly1 = min((u0 + nu) * ROWS - 1, a.H - 1);
        const int ch = a.H >> 1;
        cy0 = (ly0 & 1) ? (ly0 >> 1) : max((ly0 >> 1) - 1, 0);
        cy1 = (ly1 & 1) ? min((ly1 >> 1) + 1, ch - 1) : (ly1 >> 1);
    }
};

// The copies that stage tile `tl` (rows clamped to the frame, windows
// 16-byte aligned): cp(smem dst, global src, bytes) per contiguous piece.
template <int FAMILY, typename IN, typename CP>
__device__ __forceinline__ void f2t_copies(const F2TArgs &a, const F2TTile &tl, const F2TWindow &w, const DevFrame &f,
                                           uint8_t *st, CP &&cp)
{
    using S = F2TStage<FAMILY, IN>;
    const S sg(a.ls, a.cs, a.band);
    const int nl = tl.ly1 - tl.ly0 + 1;
    if constexpr (FAMILY == kYUV420) {
        const int nc = tl.cy1 - tl.cy0 + 1;
        if (a.whole) {
            cp(sg.luma(st, 0), row_ptr<IN>(f, 0, tl.ly0), nl * a.ls * sizeof(IN));
            cp(sg.chroma(st, 0, 0), row_ptr<IN>(f, 1, tl.cy0), nc * a.cs * sizeof(IN));
            cp(sg.chroma(st, 1, 0), row_ptr<IN>(f, 2, tl.cy0), nc * a.cs * sizeof(IN));
        } else {
            const uint32_t lb = (w.lw1 - w.lw0) * sizeof(IN), cb = (w.cw1 - w.cw0) * sizeof(IN);
            for (int r = 0; r < nl; ++r) cp(sg.luma(st, r), row_ptr<IN>(f, 0, tl.ly0 + r) + w.lw0, lb);
            for (int p = 0; p < 2; ++p)
                for (int r = 0; r < nc; ++r) cp(sg.chroma(st, p, r), row_ptr<IN>(f, p + 1, tl.cy0 + r) + w.cw0, cb);
        }
    } else {
        if (a.whole) {
            for (int p = 0; p < 3; ++p) cp(sg.plane(st, p, 0), row_ptr<IN>(f, p, tl.ly0), nl * a.ls * sizeof(IN));
        } else {
            const uint32_t lb = (w.lw1 - w.lw0) * sizeof(IN);
            for (int p = 0; p < 3; ++p)
                for (int r = 0; r < nl; ++r) cp(sg.plane(st, p, r), row_ptr<IN>(f, p, tl.ly0 + r) + w.lw0, lb);
        }
    }
}

// Stage tile t: write the consumers' view of the tile (F2THdr), then issue
// its TMA bulk copies, completing by byte count on `bar`.  t < 0: the
// end-of-work header (u0 = -1), the stage's phase completed without data.
template <int FAMILY, typename IN>
__device__ __forceinline__ void f2t_issue(const F2TArgs &a, int64_t t, uint8_t *st, uint64_t *bar, F2THdr *hdr)
{
    using S = F2TStage<FAMILY, IN>;
    if (t < 0) {
        hdr->u0 = -1;
        mbar_arrive(bar);
        return;
    }
    F2TTile tl;
    tl.set(a, t, S::ROWS);
    const DevFrame f = load_frame(a.frames + a.job_frame[tl.job]);
    F2TWindow w;
    w.set(tl.x0, tl.x1, a.W, S::G, FAMILY == kYUV420);
    *hdr = F2THdr{tl.u0, tl.nu, tl.x0, tl.x1, tl.ly0, tl.cy0, a.whole ? 0 : w.lw0, a.whole ? 0 : w.cw0};
    if (a.debug & 4) {  // experiment: no loads
        mbar_arrive(bar);
        return;
    }
    uint32_t total = 0;
    f2t_copies<FAMILY, IN>(a, tl, w, f, st, [&](void *, const void *, uint32_t bytes) { total += bytes; });
    mbar_arrive_expect_tx(bar, total);
    f2t_copies<FAMILY, IN>(a, tl, w, f, st, [&](void *dst, const void *src, uint32_t bytes) {
#ifdef NNVISR_CHECKED
        // into this stage, from inside one of the frame's planes
        NNVISR_CHECK(static_cast<uint8_t *>(dst) >= st && static_cast<uint8_t *>(dst) + bytes <= st + a.stage_bytes);
        bool inside = false;
        for (int p = 0; p < 3; ++p) {
            const int rows = (p > 0 && FAMILY == kYUV420) ? a.H >> 1 : a.H;
            const char *lo = static_cast<const char *>(f.plane[p]);
            inside |= static_cast<const char *>(src) >= lo && static_cast<const char *>(src) + bytes <= lo + rows * f.pitch[p];
        }
        NNVISR_CHECK(inside);
#endif
        bulk_g2s(dst, src, bytes, bar);
    });
}

// Warp-specialised: warps 0 .. CT/32-1 convert (consumers, CT = a.cthreads <=
// 256: one thread per 8-column group of the segment); lane 0 of the next two
// warps are the two "storers".  Per input stage k: full[k] (TMA bytes landed).
// Per output buffer b: conv[b] (every consumer warp has read tile i's stage and
// written its converted band into buffer b), ofree[b] (the bulk stores that
// read it are done).  Storer s handles tiles s, s + 2, ...: on conv[i] it
// refills tile i's stage with tile i + nst (TMA bulk copies, issued before
// tile i's stores so they do not queue behind them), frees an older output
// buffer and fans tile i out with bulk stores.  No consumer ever waits on a
// store.  Each stage's tile header (F2THdr) is written before the
// expect_tx arrive (release), so the consumers read it after their full wait
// (acquire) instead of decoding the tile index themselves.
// Output buffer layout: [channel][B*ROWS rows][sw]: with a single segment a
// channel's band rows are contiguous in the tensor too, one bulk store each.
// NARROW: a two-CTA launch with at most kNarrowCT converting threads (rows
// up to 1536 columns, e.g. 720p: 160): its register budget (2 x 256 threads)
// holds the consumer without spills, which the 320-thread bound does not.
constexpr int kNarrowCT = 192;
template <int FAMILY, typename IN, typename OUT, bool LOADER, bool YUVN, bool NARROW = false>
__global__ void __launch_bounds__(NARROW ? kNarrowCT + 64 : kThreads + (LOADER ? 96 : 64), LOADER ? 1 : 2)
    f2t_tma(const F2TArgs a)
{
    using S = F2TStage<FAMILY, IN>;
    using V8 = typename Pack<IN>::V8;
    using V4 = typename Pack<IN>::V4;
    constexpr int ROWS = S::ROWS;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem), *empty = full + kMaxStages, *ofree = empty + kMaxStages,
             *conv = ofree + kMaxOutBufs;
    F2THdr *hdr = reinterpret_cast<F2THdr *>(conv + kMaxOutBufs);
    uint8_t *stages = smem + kBarBytes;
    const int nst = a.stages, nob = a.nob, brows = a.band * ROWS;
    const S sg(a.ls, a.cs, a.band);
    OUT *obuf = reinterpret_cast<OUT *>(stages + nst * a.stage_bytes);
    int64_t *tile_of = reinterpret_cast<int64_t *>(hdr + kMaxStages);  // [kTileRing]: local tile -> launch tile
    const int CT = a.cthreads;  // converting threads (warps 0 .. CT/32-1); storers / loader follow

    if (threadIdx.x == 0) {
        for (int k = 0; k < nst; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], CT / 32);
        }
        for (int b = 0; b < nob; ++b) {
            mbar_init(&ofree[b], 1);
            mbar_init(&conv[b], CT / 32);
        }
        fence_barrier_init();
    }
    __syncthreads();  // the last CTA-wide barrier: roles split below

    // Dynamic tiles (TileSource): one thread fetches them in local order --
    // the loader (LOADER), else storer 0 for the first nst local tiles and
    // consumer thread 0 for local tile i + nst while converting tile i.  The
    // first fetch past the end gives local tile m the end-of-work header;
    // tile_of[] holds -1 from m on.  The consumers stop at m, arriving on
    // conv for m and m + 1 so both storers see the end.
    if (threadIdx.x >= CT) {
        if ((threadIdx.x & 31) != 0) return;
        if (LOADER && threadIdx.x == CT + 64) {  // ---------------- loader (LOADER variant)
            TileSource ts;
            ts.init(a.tile_counter, a.tiles);
            int k = 0;
            uint32_t rnd = 0;  // (i / nst) & 1
            for (int64_t i = 0;; ++i) {
                if (i >= nst) {  // stage k was last used by local tile i - nst
                    mbar_wait(&empty[k], rnd ^ 1u);
                    fence_proxy_async();
                }
                const int64_t t = ts.fetch();
                tile_of[i % kTileRing] = t;
                if (t < 0) tile_of[(i + 1) % kTileRing] = -1;
                NNVISR_TRACE(true, 0, i);
                f2t_issue<FAMILY, IN>(a, t, stages + k * a.stage_bytes, &full[k], &hdr[k]);
                if (t < 0) break;
                if (++k == nst) {
                    k = 0;
                    rnd ^= 1u;
                }
            }
            return;
        }
        // ---------------- storers
        // NS = a.nstorers storers (lane 0 of warps CT/32, CT/32 + 1); storer s fans out
        // tiles s, s + NS, ...  Bulk groups are per thread, so one storer
        // waiting for its own stores to drain never stalls another's issue.
        // Every destination's stores form one bulk group; eb[m] = groups
        // committed through this storer's tile i - m*NS.  The buffer of tile
        // j = i + r (r >= 1, (nob - r) % NS == 0) was last read by the
        // stores of tile j - nob, this storer's own tile `back` = (nob-r)/NS
        // tiles earlier.  back == 0: released once tile i has drained.
        // Otherwise released either BEFORE tile i is issued (release_first:
        // issue blocks while the SM's TMA unit works through earlier stores,
        // so the consumers get the buffer early) or right after (a deeper
        // store queue), once at most the groups committed since tile j - nob
        // are still reading.  A storer reaching the end-of-work tile still
        // frees buffer j (the consumers' closing arrival may wait on it).
        const int NS = a.nstorers;
        const int sidx = (threadIdx.x - CT) >> 5;
        if (sidx >= NS) return;
        if (!LOADER && sidx == 0) {
            TileSource ts;
            ts.init(a.tile_counter, a.tiles);
            bool end = false;
            for (int k = 0; k < nst; ++k) {
                const int64_t t = end ? -1 : ts.fetch();
                tile_of[k] = t;
                if (!end) f2t_issue<FAMILY, IN>(a, t, stages + k * a.stage_bytes, &full[k], &hdr[k]);
                end = t < 0;
            }
            if (end) tile_of[nst % kTileRing] = -1;
        }
        const int r = NS == 1 ? 1 : ((nob & 1) ? 1 : 2), back = (nob - r) / NS;
        int lj = -1;
        DstList dl;
        const int64_t plane = static_cast<int64_t>(a.Hp) * a.Wp;
        int ng = 0;                 // groups committed by this storer
        int eb1 = 0, eb2 = 0, eb3 = 0, eb4 = 0;  // back <= 4 (nob <= 5)
        for (int64_t i = sidx;; i += NS) {
            const int b = static_cast<int>(i % nob);
            mbar_wait(&conv[b], static_cast<uint32_t>((i / nob) & 1));
            NNVISR_TRACE(true, 4, i);
            const int64_t t = tile_of[i % kTileRing];
            const int64_t j = i + r;
            const int eb = back == 1 ? eb1 : back == 2 ? eb2 : back == 3 ? eb3 : eb4;
            if (t < 0) {  // end of work: free buffer j, drain, exit
                if (j >= nob) {
                    bulk_wait_read_le(back == 0 ? 0 : ng - eb);
                    mbar_arrive(&ofree[static_cast<int>(j % nob)]);
                }
                break;
            }
            if (!LOADER) {  // stage of tile i is free: refill it with local tile i + nst
                const int k = static_cast<int>(i % nst);
                fence_proxy_async();
                NNVISR_TRACE(true, 0, i + nst);
                f2t_issue<FAMILY, IN>(a, tile_of[(i + nst) % kTileRing], stages + k * a.stage_bytes, &full[k],
                                      &hdr[k]);
            }
            const bool rel = j >= nob;
            if (rel && back > 0 && a.release_first) {
                bulk_wait_read_le(ng - eb);
                mbar_arrive(&ofree[static_cast<int>(j % nob)]);
                NNVISR_TRACE(true, 6, i);
            }
            // fan tile i out to every (run, slot) holding its frame
            F2TTile tl;
            tl.set(a, t, ROWS);
            const int sw = tl.x1 - tl.x0, rows = tl.nu * ROWS;
            if (tl.job != lj) {
                lj = tl.job;
                dl.load(a, tl.job);
            }
            const OUT *ob = obuf + b * a.ob_elems;
            // checked builds: every bulk store reads inside this tile's output buffer
            auto s2g_ob = [&](OUT *dst, const OUT *src, uint32_t bytes) {
                NNVISR_CHECK(src >= ob && reinterpret_cast<const char *>(src) + bytes <=
                                              reinterpret_cast<const char *>(ob + a.ob_elems));
                bulk_s2g(dst, src, bytes);
            };
            const bool whole_rows = tl.x0 == 0 && sw == a.Wp;
            const int nd = (a.debug & 2) ? 0 : dl.nd;
            for (int d = 0; d < nd; ++d) {
                const int cd = dl.get(a, d);
                OUT *o = reinterpret_cast<OUT *>(a.dst + static_cast<int64_t>(cd >> 5) * a.run_stride +
                                                 static_cast<int64_t>(cd & 31) * a.slot_bytes) +
                         static_cast<int64_t>(tl.u0 * ROWS) * a.Wp + tl.x0;
                if constexpr (YUVN) {
                    // luma rows to the luma tensor; the row units' chroma rows
                    // (one per unit) to the two chroma planes of dst2
                    constexpr bool SUB = FAMILY == kYUV420;
                    const int swc = SUB ? sw >> 1 : sw;
                    if (whole_rows) {
                        s2g_ob(o, ob, rows * sw * sizeof(OUT));
                    } else {
                        for (int rr = 0; rr < rows; ++rr)
                            s2g_ob(o + static_cast<int64_t>(rr) * a.Wp, ob + rr * sw, sw * sizeof(OUT));
                    }
                    char *cb = a.dst2 + static_cast<int64_t>(cd >> 5) * a.run_stride2 +
                               static_cast<int64_t>(cd & 31) * a.slot_bytes2;
                    const OUT *oc = ob + brows * sw;
                    for (int pc = 0; pc < 2; ++pc) {
                        OUT *q = reinterpret_cast<OUT *>(cb + pc * a.cplane_bytes) +
                                 static_cast<int64_t>(tl.u0) * a.Wc + (SUB ? tl.x0 >> 1 : tl.x0);
                        const OUT *src = oc + pc * a.band * swc;
                        if (whole_rows) {
                            s2g_ob(q, src, tl.nu * swc * sizeof(OUT));
                        } else {
                            for (int rr = 0; rr < tl.nu; ++rr)
                                s2g_ob(q + static_cast<int64_t>(rr) * a.Wc, src + rr * swc, swc * sizeof(OUT));
                        }
                    }
                    bulk_commit();
                    ++ng;
                } else {
                    for (int c = 0; c < 3; ++c) {
                        if (whole_rows) {
                            s2g_ob(o + c * plane, ob + c * brows * sw, rows * sw * sizeof(OUT));
                        } else {
                            for (int rr = 0; rr < rows; ++rr)
                                s2g_ob(o + c * plane + static_cast<int64_t>(rr) * a.Wp, ob + (c * brows + rr) * sw,
                                       sw * sizeof(OUT));
                        }
                    }
                    bulk_commit();
                    ++ng;
                }
            }
            NNVISR_TRACE(true, 5, i);
            if (rel && (back == 0 || !a.release_first)) {
                bulk_wait_read_le(back == 0 ? 0 : ng - eb);
                mbar_arrive(&ofree[static_cast<int>(j % nob)]);
                NNVISR_TRACE(true, 6, i);
            }
            eb4 = eb3;
            eb3 = eb2;
            eb2 = eb1;
            eb1 = ng;
        }
        bulk_wait_all();
        return;
    }

    // ------------------------------------------------------------ consumers
    if (threadIdx.x == 0) {
        NNVISR_TRACE_CTA(0, gtimer());
        NNVISR_TRACE_CTA(2, smid());
    }
    const int cw = a.W >> 1, ch = a.H >> 1;
    const int tid = threadIdx.x;
    const bool left = FAMILY == kYUV420 && a.left;  // 4:2:0 chroma siting (reading A5)
    int k = 0, b = 0;            // stage and output buffer of tile i
    uint32_t fph = 0, bround = 0;  // full[k] wait parity; (i / nob) & 1
    TileSource ts;
    ts.init(a.tile_counter, a.tiles, nst);
    for (int64_t i = 0;; ++i) {
        uint8_t *st = stages + k * a.stage_bytes;
        OUT *ob = obuf + b * a.ob_elems;
        mbar_wait(&full[k], fph);
        NNVISR_TRACE(threadIdx.x == 0, 1, i);
        const F2THdr tl = hdr[k];
        if (tl.u0 < 0) {  // end of work at local tile i: release both storers
            for (int64_t e = i; e <= i + 1; ++e) {
                const int be = static_cast<int>(e % nob);
                if (e >= nob) mbar_wait(&ofree[be], static_cast<uint32_t>(((e / nob) & 1) ^ 1));
                __syncwarp();
                if ((threadIdx.x & 31) == 0) mbar_arrive(&conv[be]);
            }
            break;
        }
        // non-LOADER: thread 0 fetches local tile i + nst (the storer of tile
        // i stages it); the atomic's latency hides behind this tile's work
        int64_t next_t = 0;
        if (!LOADER && threadIdx.x == 0) next_t = ts.fetch();
        const int sw = tl.x1 - tl.x0;
        if (i >= nob) mbar_wait(&ofree[b], bround ^ 1u);
        NNVISR_TRACE(threadIdx.x == 0, 2, i);
        // a segment wider than kSegW (wide whole-row tiles): each thread
        // converts one 8-column group per kSegW columns
        for (int x = tl.x0 + kPx * tid; x < tl.x1; x += CT * kPx) {
        const bool fast = x + kPx <= a.W;
        if constexpr (YUVN) {
            // YUV-native tensors (NEXT-3, reading A22): no matrix, no
            // resampling: luma Y' = (16c - y_off) * y_scale, chroma
            // U = (16c - u_off) * c_scale of the unit's own chroma row, each
            // one exact integer offset and one fp32 rounding
            constexpr bool SUB = FAMILY == kYUV420;
            constexpr int NC = SUB ? 4 : kPx;
            using RowC = typename std::conditional<SUB, Row4<OUT>, Row8<OUT>>::type;
            const int swc = SUB ? sw >> 1 : sw, cx = SUB ? x >> 1 : x, cwid = SUB ? cw : a.W;
            if (x < tl.x1) {
                for (int u = 0; u < tl.nu; ++u) {
#pragma unroll
                    for (int r = 0; r < ROWS; ++r) {
                        const int yc = min((tl.u0 + u) * ROWS + r, a.H - 1);
                        const IN *L = (SUB ? sg.luma(st, yc - tl.ly0) : sg.plane(st, 0, yc - tl.ly0)) - tl.lw0;
                        int c[kPx];
                        if (fast) {
                            unpack8(ld_stage<V8>(L + x, st, a.stage_bytes), c);
                        } else {
#pragma unroll
                            for (int kk = 0; kk < kPx; ++kk) c[kk] = L[min(x + kk, a.W - 1)];
                        }
                        float v[kPx];
#pragma unroll
                        for (int kk = 0; kk < kPx; ++kk)
                            v[kk] = static_cast<float>(16 * c[kk] - a.col.y_off) * a.col.y_scale;
                        Row8<OUT> o1;
                        o1.set(v);
                        NNVISR_CHECK(ob + (u * ROWS + r) * sw + (x - tl.x0) + kPx <= ob + a.ob_elems);
                        o1.store(ob + (u * ROWS + r) * sw + (x - tl.x0));
                    }
                    const int jc = SUB ? min(tl.u0 + u, ch - 1) : min(tl.u0 + u, a.H - 1);
#pragma unroll
                    for (int pc = 0; pc < 2; ++pc) {
                        const IN *Cr = (SUB ? sg.chroma(st, pc, jc - tl.cy0) - tl.cw0
                                            : sg.plane(st, 1 + pc, jc - tl.ly0) - tl.lw0);
                        int c[NC];
                        if (fast) {
                            if constexpr (SUB) unpack4(ld_stage<V4>(Cr + cx, st, a.stage_bytes), c);
                            else unpack8(ld_stage<V8>(Cr + cx, st, a.stage_bytes), c);
                        } else {
#pragma unroll
                            for (int kk = 0; kk < NC; ++kk) c[kk] = Cr[min(cx + kk, cwid - 1)];
                        }
                        float v[NC];
#pragma unroll
                        for (int kk = 0; kk < NC; ++kk)
                            v[kk] = static_cast<float>(16 * c[kk] - a.col.u_off) * a.col.c_scale;
                        RowC oc;
                        oc.set(v);
                        NNVISR_CHECK(ob + brows * sw + (pc * a.band + u) * swc + (cx - (SUB ? tl.x0 >> 1 : tl.x0)) + NC <= ob + a.ob_elems);
                        oc.store(ob + brows * sw + (pc * a.band + u) * swc + (cx - (SUB ? tl.x0 >> 1 : tl.x0)));
                    }
                }
            }
        } else if (x < tl.x1 && !(a.debug & 1)) {
            for (int u = 0; u < tl.nu; ++u) {
                const int y0 = (tl.u0 + u) * ROWS;
                OUT *orow = ob + (u * ROWS) * sw + (x - tl.x0);
                if constexpr (FAMILY == kYUV420) {
                    if (fast && y0 + 1 < a.H) {
                        // both luma rows of the pair inside the frame (reading
                        // A5: row 2j takes 3*row j + row j-1 of chroma, row
                        // 2j+1 3*row j + row j+1, clamped; then (3/4, 1/4)
                        // horizontally).  Chroma rows j-1, j, j+1 are
                        // converted once (magic floats minus c_off/16, so the
                        // weight-16 sums come out as us - c_off exactly) and
                        // filtered vertically first.
                        const int j = y0 >> 1, i0 = x >> 1;
                        const int jr[3] = {max(j - 1, 0), j, min(j + 1, ch - 1)};
                        const float coff = kMagic + static_cast<float>(a.col.c_off >> 4);
                        float cd[2][2][kPx];  // [plane][row of the pair][column]: chroma - c_off
#pragma unroll
                        for (int p = 0; p < 2; ++p) {
                            float f[3][6];
#pragma unroll
                            for (int q = 0; q < 3; ++q) {
                                const IN *C = sg.chroma(st, p, jr[q] - tl.cy0) - tl.cw0;
                                mag4(ld_stage<V4>(C + i0, st, a.stage_bytes), &f[q][1]);
                                f[q][0] = mag(kMagicBits | C[max(i0 - 1, 0)]);
                                f[q][5] = mag(kMagicBits | C[min(i0 + 4, cw - 1)]);
#pragma unroll
                                for (int t = 0; t < 6; t += 2) {  // packed f32x2 (sm_100 FADD2 / FFMA2)
                                    const float2 d2 = __fadd2_rn(make_float2(f[q][t], f[q][t + 1]),
                                                                 make_float2(-coff, -coff));
                                    f[q][t] = d2.x;
                                    f[q][t + 1] = d2.y;
                                }
                            }
#pragma unroll
                            for (int r = 0; r < 2; ++r) {
                                float v[6];
#pragma unroll
                                for (int t = 0; t < 6; t += 2) {
                                    const float2 v2 = __ffma2_rn(make_float2(3.0f, 3.0f),
                                                                 make_float2(f[1][t], f[1][t + 1]),
                                                                 make_float2(f[r ? 2 : 0][t], f[r ? 2 : 0][t + 1]));
                                    v[t] = v2.x;
                                    v[t + 1] = v2.y;
                                }
                                if (!left) {
#pragma unroll
                                    for (int m = 0; m < 4; ++m) {
                                        const float2 h2 = __ffma2_rn(make_float2(3.0f, 3.0f),
                                                                     make_float2(v[m + 1], v[m + 1]),
                                                                     make_float2(v[m], v[m + 2]));
                                        cd[p][r][2 * m] = h2.x;
                                        cd[p][r][2 * m + 1] = h2.y;
                                    }
                                } else {  // LEFT (MPEG-2): co-sited even columns, (1/2, 1/2) odd
#pragma unroll
                                    for (int m = 0; m < 4; ++m) {
                                        cd[p][r][2 * m] = 4.0f * v[m + 1];
                                        cd[p][r][2 * m + 1] = 2.0f * (v[m + 1] + v[m + 2]);
                                    }
                                }
                            }
                        }
                        const float yoff = kMagic + static_cast<float>(a.col.y_off >> 4);
                        const float ys16 = 16.0f * a.col.y_scale;
                        const float2 yo2 = make_float2(-yoff, -yoff), ys2 = make_float2(ys16, ys16);
                        const float2 rv2 = make_float2(a.col.r_v, a.col.r_v), bu2 = make_float2(a.col.b_u, a.col.b_u);
                        const float2 gu2 = make_float2(-a.col.g_u, -a.col.g_u), gv2 = make_float2(-a.col.g_v, -a.col.g_v);
#pragma unroll
                        for (int r = 0; r < 2; ++r) {
                            float dy[kPx];
                            mag8(ld_stage<V8>(sg.luma(st, y0 + r - tl.ly0) - tl.lw0 + x, st, a.stage_bytes), dy);
                            float R[kPx], G[kPx], B[kPx];
#pragma unroll
                            for (int m = 0; m < 4; ++m) {  // pixels 2m, 2m+1 in f32x2 (same per-lane rounding)
                                const float2 dyv = __fadd2_rn(make_float2(dy[2 * m], dy[2 * m + 1]), yo2);
                                const float2 Y = __fmul2_rn(dyv, ys2);
                                const float2 du = make_float2(cd[0][r][2 * m], cd[0][r][2 * m + 1]);
                                const float2 dv = make_float2(cd[1][r][2 * m], cd[1][r][2 * m + 1]);
                                const float2 R2 = __ffma2_rn(rv2, dv, Y), B2 = __ffma2_rn(bu2, du, Y);
                                const float2 G2 = __ffma2_rn(gv2, dv, __ffma2_rn(gu2, du, Y));
                                R[2 * m] = R2.x;
                                R[2 * m + 1] = R2.y;
                                G[2 * m] = G2.x;
                                G[2 * m + 1] = G2.y;
                                B[2 * m] = B2.x;
                                B[2 * m + 1] = B2.y;
                                f2t_fix_tiny<OUT>(a.col, dyv.x, du.x, dv.x, R[2 * m], G[2 * m], B[2 * m]);
                                f2t_fix_tiny<OUT>(a.col, dyv.y, du.y, dv.y, R[2 * m + 1], G[2 * m + 1], B[2 * m + 1]);
                            }
                            Row8<OUT> o3[3];
                            o3[0].set(R);
                            o3[1].set(G);
                            o3[2].set(B);
#pragma unroll
                            for (int c = 0; c < 3; ++c) {
#ifdef NNVISR_CHECKED
                                NNVISR_CHECK(orow + (c * brows + r) * sw >= ob && orow + (c * brows + r) * sw + kPx <= ob + a.ob_elems);
#endif
                                o3[c].store(orow + (c * brows + r) * sw);
                            }
                        }
                        continue;
                    }
                }
#pragma unroll
                for (int r = 0; r < ROWS; ++r) {
                    const int yc = min(y0 + r, a.H - 1);
                    int ys[kPx], us[kPx], vs[kPx];
                    if constexpr (FAMILY == kYUV420) {
                        // ragged right edge or padding rows: per-sample clamped taps
                        const IN *L = sg.luma(st, yc - tl.ly0) - tl.lw0;
                        const IN *Cn[2] = {sg.chroma(st, 0, chroma_near(yc) - tl.cy0) - tl.cw0,
                                           sg.chroma(st, 1, chroma_near(yc) - tl.cy0) - tl.cw0};
                        const IN *Cf[2] = {sg.chroma(st, 0, chroma_far(yc, ch) - tl.cy0) - tl.cw0,
                                           sg.chroma(st, 1, chroma_far(yc, ch) - tl.cy0) - tl.cw0};
#pragma unroll
                        for (int kk = 0; kk < kPx; ++kk) {
                            const int xc = min(x + kk, a.W - 1);
                            ys[kk] = 16 * L[xc];
                            const int in_ = xc >> 1;
                            if (!left) {
                                const int if_ = (xc & 1) ? min(in_ + 1, cw - 1) : max(in_ - 1, 0);
                                us[kk] = 9 * Cn[0][in_] + 3 * Cn[0][if_] + 3 * Cf[0][in_] + Cf[0][if_];
                                vs[kk] = 9 * Cn[1][in_] + 3 * Cn[1][if_] + 3 * Cf[1][in_] + Cf[1][if_];
                            } else {  // LEFT: co-sited column xc/2 (even xc) or the mean of xc/2 and xc/2+1
                                const int i1 = (xc & 1) ? min(in_ + 1, cw - 1) : in_;
                                us[kk] = 2 * (3 * (Cn[0][in_] + Cn[0][i1]) + Cf[0][in_] + Cf[0][i1]);
                                vs[kk] = 2 * (3 * (Cn[1][in_] + Cn[1][i1]) + Cf[1][in_] + Cf[1][i1]);
                            }
                        }
                    } else {
                        const IN *P0 = sg.plane(st, 0, yc - tl.ly0) - tl.lw0,
                                 *P1 = sg.plane(st, 1, yc - tl.ly0) - tl.lw0,
                                 *P2 = sg.plane(st, 2, yc - tl.ly0) - tl.lw0;
                        if (fast) {
                            unpack8(ld_stage<V8>(P0 + x, st, a.stage_bytes), ys);
                            unpack8(ld_stage<V8>(P1 + x, st, a.stage_bytes), us);
                            unpack8(ld_stage<V8>(P2 + x, st, a.stage_bytes), vs);
                        } else {
#pragma unroll
                            for (int kk = 0; kk < kPx; ++kk) {
                                const int xc = min(x + kk, a.W - 1);
                                ys[kk] = P0[xc];
                                us[kk] = P1[xc];
                                vs[kk] = P2[xc];
                            }
                        }
#pragma unroll
                        for (int kk = 0; kk < kPx; ++kk) {
                            ys[kk] *= 16;
                            us[kk] *= 16;
                            vs[kk] *= 16;
                        }
                    }
                    Row8<OUT> o3[3];
                    f2t_row<FAMILY, OUT>(a.col, ys, us, vs, o3);
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
#ifdef NNVISR_CHECKED
                        NNVISR_CHECK(orow + (c * brows + r) * sw >= ob && orow + (c * brows + r) * sw + kPx <= ob + a.ob_elems);
#endif
                        o3[c].store(orow + (c * brows + r) * sw);
                    }
                }
            }
        }
        }  // column groups
        fence_proxy_async();  // generic-proxy smem writes -> visible to the bulk stores
        if (!LOADER && threadIdx.x == 0) {
            tile_of[(i + nst) % kTileRing] = next_t;
            if (next_t < 0) tile_of[(i + nst + 1) % kTileRing] = -1;
        }
        __syncwarp();
        NNVISR_TRACE(threadIdx.x == 0, 3, i);
        if ((threadIdx.x & 31) == 0) {
            if (LOADER) mbar_arrive(&empty[k]);
            mbar_arrive(&conv[b]);
        }
        if (++k == nst) {
            k = 0;
            fph ^= 1u;
        }
        if (++b == nob) {
            b = 0;
            bround ^= 1u;
        }
    }
    if (threadIdx.x == 0) NNVISR_TRACE_CTA(1, gtimer());
}

// ------------------------------------------------------------------ t2f
// Stage layout (values of TIN): [ROWS][3 channels][segw], segw = the launch's
// (equal) segment width.  The producer writes each stage's T2FHdr before its
// expect_tx arrive, so the consumers read the tile's output frame, rows and
// columns after their full wait instead of decoding the tile index.
struct T2FHdr {
    int job, y0, x0, x1;
};

// Staged row (r, c): stride segw + lpad values, the segment's first column at
// offset lpad (LEFT siting stages the column left of the segment there).
template <int FAMILY, typename TIN>
__device__ __forceinline__ TIN *t2f_row_ptr(uint8_t *st, int segw, int lpad, int r, int c)
{
    return reinterpret_cast<TIN *>(st) + (r * 3 + c) * (segw + lpad) + lpad;
}

// Stage tile t; t < 0: write the end-of-work header (job -1) and complete
// the stage's phase without data.
template <int FAMILY, typename TIN>
__device__ __forceinline__ void t2f_issue(const T2FArgs &a, int64_t t, uint8_t *st, uint64_t *bar, T2FHdr *hdr)
{
    constexpr int ROWS = FAMILY == kYUV420 ? 2 : 1;
    if (t < 0) {
        hdr->job = -1;
        mbar_arrive(bar);
        return;
    }
    int job, ru, x0;
    decode_tile(t, a.rowunits, a.nseg, a.segw, job, ru, x0);
    const int x1 = min(x0 + a.segw, a.Wo);
    int tup, o;
    t2f_job(a, job, tup, o);
    *hdr = T2FHdr{job, ru * ROWS, x0, x1};
    const int64_t plane = a.th * a.tw;
    const TIN *src = reinterpret_cast<const TIN *>(a.src + static_cast<int64_t>(tup) * a.tensor_stride) +
                     static_cast<int64_t>(3 * o) * plane + static_cast<int64_t>(ru * ROWS) * a.tw + x0;
    // LEFT siting: also the lpad values left of the segment (x0 > 0; 16 bytes);
    // a ragged end (output width not a multiple of 8) is copied up to the next
    // 16 bytes, inside the tensor row (its width is a 16-byte multiple)
    const int pre = x0 > 0 ? a.lpad : 0;
    constexpr int G = 16 / sizeof(TIN);
    const int xe = (x1 + G - 1) / G * G;
    const uint32_t bytes = (xe - x0 + pre) * sizeof(TIN);
    mbar_arrive_expect_tx(bar, ROWS * 3 * bytes);
#pragma unroll
    for (int r = 0; r < ROWS; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
#ifdef NNVISR_CHECKED
            {  // into this stage, from inside output slot o's three channels of tuple tup
                const uint8_t *d = reinterpret_cast<const uint8_t *>(t2f_row_ptr<FAMILY, TIN>(st, a.segw, a.lpad, r, c) - pre);
                const TIN *q = src + c * plane + r * a.tw - pre;
                const TIN *lo = reinterpret_cast<const TIN *>(a.src + static_cast<int64_t>(tup) * a.tensor_stride) +
                                static_cast<int64_t>(3 * o) * plane;
                NNVISR_CHECK(d >= st && d + bytes <= st + a.stage_bytes);
                NNVISR_CHECK(q >= lo && reinterpret_cast<const char *>(q) + bytes <=
                                            reinterpret_cast<const char *>(lo + 3 * plane));
            }
#endif
            bulk_g2s(t2f_row_ptr<FAMILY, TIN>(st, a.segw, a.lpad, r, c) - pre, src + c * plane + r * a.tw - pre, bytes,
                     bar);
        }
}

// Warp-specialised like f2t_tma: a.cthreads consumer threads (segw / 8,
// rounded up to whole warps) convert and store with st.global; lane 0 of the
// last warp keeps the stages full.
template <int FAMILY, typename OS, typename TIN, typename AR>
__global__ void __launch_bounds__(kThreads + 32, (FAMILY == kYUV420 && sizeof(AR) == 8) ? 2 : 3) t2f_tma(const T2FArgs a)
{
    constexpr int ROWS = FAMILY == kYUV420 ? 2 : 1;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem), *empty = full + kMaxStages;
    T2FHdr *hdr = reinterpret_cast<T2FHdr *>(empty + kMaxStages);
    uint8_t *stages = smem + kBarBytes;
    const int nst = a.stages, nct = a.cthreads;

    if (threadIdx.x == 0) {
        for (int k = 0; k < nst; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], nct / 32);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (threadIdx.x >= nct) {  // ---------------- producer warp
        if (threadIdx.x != nct) return;
        TileSource ts;
        ts.init(a.tile_counter, a.tiles);
        // stage k of local tile i; stop after staging the end-of-work header
        int k = 0;
        uint32_t rnd = 0;  // (i / nst) & 1
        for (int64_t i = 0;; ++i) {
            if (i >= nst) {  // stage k was last used by local tile i - nst
                mbar_wait(&empty[k], rnd ^ 1u);
                fence_proxy_async();
            }
            const int64_t t = ts.fetch();
            t2f_issue<FAMILY, TIN>(a, t, stages + k * a.stage_bytes, &full[k], &hdr[k]);
            if (t < 0) break;
            if (++k == nst) {
                k = 0;
                rnd ^= 1u;
            }
        }
        return;
    }

    // ------------------------------------------------------------ consumers
    const T2FConst<AR> c(a.col);
    int cj = -1;
    DevFrame f;
    const int xo = kPx * threadIdx.x;  // column within the segment
    int k = 0;
    uint32_t fph = 0;
    for (;;) {
        uint8_t *st = stages + k * a.stage_bytes;
        mbar_wait(&full[k], fph);
        const T2FHdr h = hdr[k];
        if (h.job < 0) break;
        if (h.job != cj) {
            cj = h.job;
            f = load_frame(a.out + cj);
        }
        if (h.x0 + xo < h.x1) {
            const int x = h.x0 + xo;
            // the last group of a ragged row stores only its valid columns
            const int nv = min(kPx, h.x1 - x);
            const bool vec = a.vec_out && nv == kPx;
            AR sb[4], sr[4];
            if (FAMILY == kYUV420 && a.lpad) {
                // LEFT (MPEG-2) siting: per row the [1,2,1] taps need B-Y', R-Y'
                // of column x-1 (column 0 at x = 0), staged left of the segment
                const int xl = x > 0 ? xo - 1 : xo;
#pragma unroll
                for (int r = 0; r < ROWS; ++r) {
                    const TIN *p0 = t2f_row_ptr<FAMILY, TIN>(st, a.segw, a.lpad, r, 0);
                    const TIN *p1 = t2f_row_ptr<FAMILY, TIN>(st, a.segw, a.lpad, r, 1);
                    const TIN *p2 = t2f_row_ptr<FAMILY, TIN>(st, a.segw, a.lpad, r, 2);
                    const AR r_ = tload1(p0 + xl), g_ = tload1(p1 + xl), b_ = tload1(p2 + xl);
                    const AR Yl = fma_(c.kb, b_ - g_, fma_(c.kr, r_ - g_, g_));
                    float R[kPx], G[kPx], B[kPx];
                    tload8(p0 + xo, R);
                    tload8(p1 + xo, G);
                    tload8(p2 + xo, B);
                    t2f_row<FAMILY, OS, AR, true>(c, a.col, f, x, h.y0 + r, r, R, G, B, nv, vec, sb, sr, b_ - Yl,
                                                  r_ - Yl);
                }
                if constexpr (FAMILY == kYUV420) t2f_chroma420<OS, AR, true>(c, f, x, h.y0, sb, sr, nv, vec);
            } else {
#pragma unroll
                for (int r = 0; r < ROWS; ++r) {
                    float R[kPx], G[kPx], B[kPx];
                    tload8(t2f_row_ptr<FAMILY, TIN>(st, a.segw, a.lpad, r, 0) + xo, R);
                    tload8(t2f_row_ptr<FAMILY, TIN>(st, a.segw, a.lpad, r, 1) + xo, G);
                    tload8(t2f_row_ptr<FAMILY, TIN>(st, a.segw, a.lpad, r, 2) + xo, B);
                    t2f_row<FAMILY, OS, AR>(c, a.col, f, x, h.y0 + r, r, R, G, B, nv, vec, sb, sr);
                }
                if constexpr (FAMILY == kYUV420) t2f_chroma420<OS, AR>(c, f, x, h.y0, sb, sr, nv, vec);
            }
        }
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[k]);
        if (++k == nst) {
            k = 0;
            fph ^= 1u;
        }
    }
}

// ------------------------------------------------------------------ t2f, YUV-native tensors
// NEXT-3 (§3.1, reading A22): the network's output is a
// luma tensor [M][th][tw] and a chroma tensor [2M][thc][twc]; step B4 only
// (scale, RNE, clamp).  Same pipeline as t2f_tma; a stage holds the tile's
// ROWS luma rows and its chroma row of each plane (4:2:0: half width, the
// row unit's chroma row):  [ROWS][segw] luma | [2][segwc] chroma.
template <int FAMILY, typename TIN>
__device__ __forceinline__ void t2f_yuv_issue(const T2FArgs &a, int64_t t, uint8_t *st, uint64_t *bar, T2FHdr *hdr)
{
    constexpr bool SUB = FAMILY == kYUV420;
    constexpr int ROWS = SUB ? 2 : 1;
    if (t < 0) {
        hdr->job = -1;
        mbar_arrive(bar);
        return;
    }
    int job, ru, x0;
    decode_tile(t, a.rowunits, a.nseg, a.segw, job, ru, x0);
    const int x1 = min(x0 + a.segw, a.Wo);
    int tup, o;
    t2f_job(a, job, tup, o);
    *hdr = T2FHdr{job, ru * ROWS, x0, x1};
    const int segwc = SUB ? a.segw >> 1 : a.segw;
    const int64_t lplane = a.th * a.tw, cplane = a.thc * a.twc;
    const TIN *ls = reinterpret_cast<const TIN *>(a.src + static_cast<int64_t>(tup) * a.tensor_stride) +
                    static_cast<int64_t>(o) * lplane + static_cast<int64_t>(ru * ROWS) * a.tw + x0;
    const int cy = SUB ? ru : ru * ROWS, cx0 = SUB ? x0 >> 1 : x0;
    const TIN *cs = reinterpret_cast<const TIN *>(a.src2 + static_cast<int64_t>(tup) * a.tensor_stride2) +
                    static_cast<int64_t>(2 * o) * cplane + static_cast<int64_t>(cy) * a.twc + cx0;
    const uint32_t lb = (x1 - x0) * sizeof(TIN), cb = (SUB ? (x1 - x0) >> 1 : x1 - x0) * sizeof(TIN);
    mbar_arrive_expect_tx(bar, ROWS * lb + 2 * cb);
    TIN *sv = reinterpret_cast<TIN *>(st);
#ifdef NNVISR_CHECKED
    {  // into this stage, from inside the slot's luma plane / two chroma planes
        const TIN *l0 = reinterpret_cast<const TIN *>(a.src + static_cast<int64_t>(tup) * a.tensor_stride) +
                        static_cast<int64_t>(o) * lplane;
        const TIN *c0 = reinterpret_cast<const TIN *>(a.src2 + static_cast<int64_t>(tup) * a.tensor_stride2) +
                        static_cast<int64_t>(2 * o) * cplane;
        NNVISR_CHECK(reinterpret_cast<const uint8_t *>(sv + ROWS * a.segw + 2 * segwc) <= st + a.stage_bytes);
        NNVISR_CHECK(ls >= l0 && reinterpret_cast<const char *>(ls + (ROWS - 1) * a.tw) + lb <=
                                     reinterpret_cast<const char *>(l0 + lplane));
        NNVISR_CHECK(cs >= c0 && reinterpret_cast<const char *>(cs + cplane) + cb <=
                                     reinterpret_cast<const char *>(c0 + 2 * cplane));
    }
#endif
#pragma unroll
    for (int r = 0; r < ROWS; ++r) bulk_g2s(sv + r * a.segw, ls + r * a.tw, lb, bar);
#pragma unroll
    for (int p = 0; p < 2; ++p) bulk_g2s(sv + ROWS * a.segw + p * segwc, cs + p * cplane, cb, bar);
}

template <int FAMILY, typename OS, typename TIN, typename AR>
__global__ void __launch_bounds__(kThreads + 32, (FAMILY == kYUV420 && sizeof(AR) == 8) ? 2 : 3)
    t2f_yuv_tma(const T2FArgs a)
{
    constexpr bool SUB = FAMILY == kYUV420;
    constexpr int ROWS = SUB ? 2 : 1, NC = SUB ? 4 : 8;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem), *empty = full + kMaxStages;
    T2FHdr *hdr = reinterpret_cast<T2FHdr *>(empty + kMaxStages);
    uint8_t *stages = smem + kBarBytes;
    const int nst = a.stages, nct = a.cthreads;
    if (threadIdx.x == 0) {
        for (int k = 0; k < nst; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], nct / 32);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (threadIdx.x >= nct) {  // ---------------- producer lane
        if (threadIdx.x != nct) return;
        TileSource ts;
        ts.init(a.tile_counter, a.tiles);
        int k = 0;
        uint32_t rnd = 0;
        for (int64_t i = 0;; ++i) {
            if (i >= nst) {
                mbar_wait(&empty[k], rnd ^ 1u);
                fence_proxy_async();
            }
            const int64_t t = ts.fetch();
            t2f_yuv_issue<FAMILY, TIN>(a, t, stages + k * a.stage_bytes, &full[k], &hdr[k]);
            if (t < 0) break;
            if (++k == nst) {
                k = 0;
                rnd ^= 1u;
            }
        }
        return;
    }

    // ------------------------------------------------------------ consumers
    const T2FConst<AR> c(a.col);
    const int segwc = SUB ? a.segw >> 1 : a.segw;
    int cj = -1;
    DevFrame f;
    const int xo = kPx * threadIdx.x;
    int k = 0;
    uint32_t fph = 0;
    for (;;) {
        const TIN *sv = reinterpret_cast<const TIN *>(stages + k * a.stage_bytes);
        mbar_wait(&full[k], fph);
        const T2FHdr h = hdr[k];
        if (h.job < 0) break;
        if (h.job != cj) {
            cj = h.job;
            f = load_frame(a.out + cj);
        }
        if (h.x0 + xo < h.x1) {
            const int x = h.x0 + xo;
            // luma: code = rne(clamp(Y' * ys + yo))
#pragma unroll
            for (int r = 0; r < ROWS; ++r) {
                float v[kPx];
                tload8(sv + r * a.segw + xo, v);
                uint32_t q[kPx];
#pragma unroll
                for (int kk = 0; kk < kPx; ++kk) q[kk] = quant_direct(static_cast<AR>(v[kk]), c.yd, c.yod, c.maxc);
                store_samples8(row_ptr_w<OS>(f, 0, h.y0 + r) + x, q);
            }
            // chroma: code = rne(clamp(U * cs + (co - cs/2)))  (reading A22)
            const int cxo = SUB ? xo >> 1 : xo, cy = SUB ? h.y0 >> 1 : h.y0, cx = SUB ? x >> 1 : x;
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                const TIN *cp_ = sv + ROWS * a.segw + p * segwc + cxo;
                uint32_t q[NC];
                if constexpr (NC == 8) {
                    float v[8];
                    tload8(cp_, v);
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) q[kk] = quant_direct(static_cast<AR>(v[kk]), c.csd, c.co2d, c.maxc);
                    store_samples8(row_ptr_w<OS>(f, 1 + p, cy) + cx, q);
                } else {
                    float v[4];
                    tload4s(cp_, v);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) q[kk] = quant_direct(static_cast<AR>(v[kk]), c.csd, c.co2d, c.maxc);
                    store_samples4(row_ptr_w<OS>(f, 1 + p, cy) + cx, q);
                }
            }
        }
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[k]);
        if (++k == nst) {
            k = 0;
            fph ^= 1u;
        }
    }
}

// ------------------------------------------------------------------ launch
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

// Tuning knobs for experiments and sweeps (NNVISR_F2T_* / NNVISR_T2F_*,
// DESIGN.md §6): read at each launch; unset = the built-in choice.
int env_int(const char *name, int dflt)
{
    const char *v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

// Dynamic smem = mbarriers | `stages` input stages | `extra` bytes (f2t: two
// output staging buffers).  Stages: `default_stages` (tools/sweep_t2f.sh on
// B200, profiles/r01/t2f_sweep.txt), else as many as fit in `budget`.
template <typename K, typename A>
cudaError_t launch_tma(K kernel, A a, int vals_per_col, int elem, int budget, int default_stages, cudaStream_t s)
{
    if (a.tiles <= 0) return cudaSuccess;
    // equal segments of a multiple of 32 columns (<= 2048): no thin tail tile;
    // a stage holds one tile's rows x 3 channels x segw values, and the
    // consumer threads are the tile's 8-column groups (whole warps)
    a.segw = std::min(kSegW, ((a.Wo + a.nseg - 1) / a.nseg + 31) / 32 * 32);
    a.cthreads = std::min(kThreads, (a.segw / kPx + 31) / 32 * 32);
    a.stage_bytes = (vals_per_col * (a.segw + a.lpad) * elem + 127) / 128 * 128;
    budget = env_int("NNVISR_T2F_SMEM_KB", budget / 1024) * 1024;
    a.stages = env_int("NNVISR_T2F_STAGES", default_stages);
    if (a.stages <= 0) a.stages = budget / a.stage_bytes;
    a.stages = std::max(2, std::min(kMaxStages, a.stages));
    const int smem = kBarBytes + a.stages * a.stage_bytes;
    const int block = a.cthreads + 32;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem);
    if (e != cudaSuccess) return e;
    const int grid = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>(a.tiles, static_cast<int64_t>(sms()) * std::max(per_sm, 1))));
    kernel<<<grid, block, smem, s>>>(a);
    return cudaGetLastError();
}

// f2t smem: mbarriers | stages x input stage | nob x output buffer.  Sized at
// run time from the segment width min(2048, Wp), to keep two CTAs per SM
// (<= 112 KB each) with 3 output buffers where they fit (more bulk stores in
// flight), else 2.
template <int FAMILY, typename IN, typename OUT, bool YUVN>
cudaError_t f2t_tma_launch(F2TArgs a, cudaStream_t s)
{
    using S = F2TStage<FAMILY, IN>;
    constexpr int ROWS = S::ROWS;
    if (a.tiles <= 0) return cudaSuccess;
    // segment width: kSegW (the host's nseg), or -- wide mode, frames up to
    // 2 x kSegW wide -- the whole padded row in one tile (whole-row copies and
    // stores; each consumer thread takes two column groups)
    const int64_t jobs_ = a.tiles / ((int64_t)a.rowunits * a.nseg);
    // (4:2:0 only: measured +5% at 4K; 4:4:4 fp32 tiles are faster split)
    int segw = 0;
    auto stage_bytes = [&](int B) { return (S(a.ls, a.cs, B).bytes() + 127) / 128 * 128; };
    // RGB: 3 planes of the band's rows; YUV-native: the luma rows plus the
    // units' two chroma rows (half width in 4:2:0)
    constexpr int kObRows = YUVN ? (FAMILY == kYUV420 ? ROWS + 1 : ROWS + 2) : 3 * ROWS;
    auto ob_bytes = [&](int B) { return (kObRows * B * segw * (int)sizeof(OUT) + 127) / 128 * 128; };
    auto segment = [&](bool wide) {
        a.fsegw = wide ? (a.Wp + 31) / 32 * 32 : kSegW;
        a.nseg = (a.Wp + a.fsegw - 1) / a.fsegw;
        a.tiles = jobs_ * a.rowunits * a.nseg;
        segw = std::min(a.fsegw, (a.Wp + 31) / 32 * 32);
        const int lcap = (segw + 2 * S::G - 1) / (2 * S::G) * (2 * S::G);  // ccap*sizeof(IN) stays 16-byte aligned
        const int ccap = lcap / 2 + 2 * S::G;
        // whole rows: one segment, and every bound frame's pitches are the staged strides
        const int sb = sizeof(IN);
        const bool whole = a.nseg == 1 && a.pitch_y > 0 && a.pitch_y % 16 == 0 && a.pitch_y / sb <= 4 * lcap &&
                           (FAMILY != kYUV420 || (a.pitch_c > 0 && a.pitch_c % 16 == 0));
        a.whole = whole;
        a.ls = whole ? a.pitch_y / sb : lcap;
        a.cs = whole ? (FAMILY == kYUV420 ? a.pitch_c / sb : a.ls) : ccap;
    };
    constexpr int kMaxSmem = 227 * 1024;
    const bool wide = env_int("NNVISR_F2T_WIDE", FAMILY == kYUV420 ? 1 : 0) && a.Wp > kSegW && a.Wp <= 2 * kSegW;
    segment(wide);
    // a whole-row tile must fit one stage and two output buffers of a single
    // row unit (16-bit fp32 4:2:0 rows near 4096 columns do not): else segments
    if (wide && kBarBytes + stage_bytes(1) + 2 * ob_bytes(1) > kMaxSmem) segment(false);
    // band height and buffering, from the tools/sweep_f2t.sh sweep on B200
    // (profiles/r01/f2t_sweep.txt): bands of 2 row units with 3 output buffers
    // for whole-row frames and 4:4:4; single row units for 4:2:0 frames wider
    // than one 2048-column segment (per-row copies, chroma halo rows)
    // Low fan-out launches (store mode, Fig. 1 slots: <= 2 destinations per
    // frame) are bound by the conversion itself: when bands of 2 would leave
    // one CTA per SM they take single row units, so two CTAs (16 converting
    // warps) share an SM.
    constexpr int kSmSmem = 228 * 1024, kCtaReserve = 1024;
    auto fits_two = [&](int B) {
        return 2 * (kBarBytes + 2 * stage_bytes(B) + 2 * ob_bytes(B) + kCtaReserve) <= kSmSmem;
    };
    const bool low_fanout = a.dests > 0 && a.dests <= 2 * a.jobs;
    int B = env_int("NNVISR_F2T_BAND", 0);
    if (B <= 0) {
        B = ((FAMILY == kYUV420 && (a.nseg > 1 || a.fsegw > kSegW)) || (low_fanout && !fits_two(2))) ? 1 : 2;
        // YUV-native output buffers are half the RGB ones in 4:2:0: bands of
        // 4 row units still fit two CTAs per SM (measured +12% at 720p)
        if (YUVN && B == 2 && fits_two(4)) B = 4;
    }
    a.band = std::max(1, std::min(B, a.rowunits));
    const int bands = (a.rowunits + a.band - 1) / a.band;
    a.tiles = a.tiles / ((int64_t)a.rowunits * a.nseg) * bands * a.nseg;  // jobs * bands * nseg
    a.stage_bytes = stage_bytes(a.band);
    a.ob_elems = ob_bytes(a.band) / (int)sizeof(OUT);
    // Two pipeline shapes, from the B200 sweeps (profiles/r01/f2t_sweep.txt):
    //  * two CTAs per SM when 2 stages + 2 output buffers fit in half the
    //    SM's shared memory (4K 4:2:0 split into 2 segments, 720p): the two
    //    storers also issue the loads (10 warps: 96 registers) and release
    //    the next output buffer before issuing a tile;
    //  * else one CTA per SM (1080p whole rows, 4K 4:4:4 fp32): a dedicated
    //    loader warp, 3 output buffers, release after issuing (a deeper
    //    store queue).
    const bool two = fits_two(a.band);
    a.stages = env_int("NNVISR_F2T_STAGES", 2);
    a.nob = env_int("NNVISR_F2T_NOB", (two || a.fsegw > kSegW) ? 2 : 3);
    a.stages = std::max(1, std::min(kMaxStages, a.stages));
    a.nob = std::max(2, std::min(5, a.nob));
    // never exceed the 227 KB a CTA may use: shed output buffers, then band rows
    while (kBarBytes + a.stages * a.stage_bytes + a.nob * ob_bytes(a.band) > kMaxSmem) {
        if (a.nob > 2) --a.nob;
        else if (a.stages > 1) --a.stages;
        else if (a.band > 1) {
            --a.band;
            a.stage_bytes = stage_bytes(a.band);
            a.ob_elems = ob_bytes(a.band) / (int)sizeof(OUT);
        } else break;
    }
    a.tiles = a.tiles / bands * ((a.rowunits + a.band - 1) / a.band);
    const int smem = kBarBytes + a.stages * a.stage_bytes + a.nob * ob_bytes(a.band);
    const bool fits2 = 2 * (smem + kCtaReserve) <= kSmSmem;
    a.nstorers = std::max(1, std::min(2, env_int("NNVISR_F2T_STORERS", 2)));
    // converting threads: one per 8-column group of a single-segment row
    // (a 1280-column row: 160 -- no idle warps; measured +1-3% at 720p), else
    // kThreads (segments of kSegW columns, or wide tiles with two groups per
    // thread).  NNVISR_F2T_CT raises it (experiments).
    {
        const int fit = (a.nseg == 1 && a.fsegw <= kSegW) ? std::min(kThreads, (a.Wp / kPx + 31) / 32 * 32) : kThreads;
        a.cthreads = std::max(fit, std::min(kThreads, (env_int("NNVISR_F2T_CT", 0) + 31) / 32 * 32));
    }
    a.release_first = env_int("NNVISR_F2T_RELFIRST", fits2 ? 1 : 0);
    // experiment switches (NNVISR_F2T_DEBUG: 1 no conversion, 2 no stores, 4 no
    // loads, 8 timeline, 16 short buffers) exist only in experiment, trace and
    // checked builds: the product library always converts, loads and stores
#if defined(NNVISR_EXPERIMENTS) || defined(NNVISR_F2T_TRACE) || defined(NNVISR_CHECKED)
    a.debug = env_int("NNVISR_F2T_DEBUG", 0);
#else
    a.debug = 0;
#endif
#ifdef NNVISR_CHECKED
    if (a.debug & 16) a.ob_elems -= 8;  // negative control: buffers too short (the checked build must trap)
#endif
    int loader = env_int("NNVISR_F2T_LOADER", fits2 ? 0 : 1);
    const bool narrow = !loader && a.cthreads <= kNarrowCT;
    auto kernel = loader ? f2t_tma<FAMILY, IN, OUT, true, YUVN>
                         : narrow ? f2t_tma<FAMILY, IN, OUT, false, YUVN, true> : f2t_tma<FAMILY, IN, OUT, false, YUVN>;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    const int block = a.cthreads + (loader ? 96 : 64);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem);
    if (e != cudaSuccess) return e;
    const int grid = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>(a.tiles, static_cast<int64_t>(sms()) * std::max(per_sm, 1))));
    static uint64_t *trace_buf = nullptr;
    constexpr size_t kTraceBytes = (2 * kTraceEvents * kTraceTiles + 3 * kTraceCtas) * sizeof(uint64_t);
    if (a.debug & 8) {
        if (!trace_buf) cudaMalloc(&trace_buf, kTraceBytes);
        cudaMemsetAsync(trace_buf, 0, kTraceBytes, s);
        a.trace = trace_buf;
    }
    kernel<<<grid, block, smem, s>>>(a);
    static int traced_launch = 0;  // NNVISR_F2T_TRACE_LAUNCH = k: dump only the k-th traced launch
    bool dump = false;
    if ((a.debug & 8) && std::getenv("NNVISR_F2T_TRACE")) {
        const int k = traced_launch++;
        dump = k == env_int("NNVISR_F2T_TRACE_LAUNCH", k);
    }
    if (dump) {  // dump the launch's timeline (experiments only)
        std::vector<uint64_t> h(kTraceBytes / sizeof(uint64_t));
        cudaMemcpyAsync(h.data(), trace_buf, kTraceBytes, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        if (FILE *fp = std::fopen(std::getenv("NNVISR_F2T_TRACE"), "w")) {
            std::fprintf(fp, "# stages %d nob %d band %d stage_bytes %d tiles %lld grid %d\n", a.stages, a.nob, a.band, a.stage_bytes, (long long)a.tiles, grid);
            for (int c = 0; c < 2; ++c)
                for (int i = 0; i < kTraceTiles; ++i) {
                    std::fprintf(fp, "%d %d", c, i);
                    for (int ev = 0; ev < kTraceEvents; ++ev)
                        std::fprintf(fp, " %llu", (unsigned long long)h[(c * kTraceEvents + ev) * kTraceTiles + i]);
                    std::fprintf(fp, "\n");
                }
            for (int c = 0; c < grid && c < kTraceCtas; ++c) {
                const uint64_t *q = &h[2 * kTraceEvents * kTraceTiles + 3 * c];
                std::fprintf(fp, "cta %d %llu %llu %llu\n", c, (unsigned long long)q[0], (unsigned long long)q[1],
                             (unsigned long long)q[2]);
            }
            std::fclose(fp);
        }
    }
    return cudaGetLastError();
}

template <int FAMILY, bool YUVN = false>
cudaError_t f2t_tma_dispatch(int bits, int dtype, const F2TArgs &a, cudaStream_t s)
{
    if (bits == 8) {
        if (dtype == kF16) return f2t_tma_launch<FAMILY, uint8_t, __half, YUVN>(a, s);
        return f2t_tma_launch<FAMILY, uint8_t, float, YUVN>(a, s);
    }
    if (dtype == kF16) return f2t_tma_launch<FAMILY, uint16_t, __half, YUVN>(a, s);
    return f2t_tma_launch<FAMILY, uint16_t, float, YUVN>(a, s);
}

template <int FAMILY>
cudaError_t t2f_tma_dispatch(int bits, int dtype, const T2FArgs &a, cudaStream_t s)
{
    // input stages: NNVISR_T2F_STAGES, else as many as fit in 50 KB (two at
    // 1080p/4K, three at 720p; tools/sweep.sh t2f on B200, profiles/r01/t2f_sweep2.txt)
    constexpr int R = FAMILY == kYUV420 ? 2 : 1, kBudget = 50 * 1024;
    const int st = env_int("NNVISR_T2F_STAGES", 0);
    T2FArgs b = a;
    b.lpad = (FAMILY == kYUV420 && a.left) ? 16 / (dtype == kF16 ? 2 : 4) : 0;  // LEFT: 16 bytes left of each row
    if (bits == 8) {
        if (dtype == kF16) return launch_tma(t2f_tma<FAMILY, uint8_t, __half, float>, b, 3 * R, 2, kBudget, st, s);
        return launch_tma(t2f_tma<FAMILY, uint8_t, float, float>, b, 3 * R, 4, kBudget, st, s);
    }
    if (bits == 10) {
        if (dtype == kF16) return launch_tma(t2f_tma<FAMILY, uint16_t, __half, float>, b, 3 * R, 2, kBudget, st, s);
        return launch_tma(t2f_tma<FAMILY, uint16_t, float, float>, b, 3 * R, 4, kBudget, st, s);
    }
    if (dtype == kF16) return launch_tma(t2f_tma<FAMILY, uint16_t, __half, double>, b, 3 * R, 2, kBudget, st, s);
    return launch_tma(t2f_tma<FAMILY, uint16_t, float, double>, b, 3 * R, 4, kBudget, st, s);
}

template <int FAMILY>
cudaError_t t2f_yuv_tma_dispatch(int bits, int dtype, const T2FArgs &a, cudaStream_t s)
{
    // values per column: ROWS luma + 2 chroma (halved for 4:2:0); stages fitting
    // 30 KB (2-3; B200 sweep: 720p 5.9 -> 6.5 TB/s against 50 KB)
    constexpr int V = 3, kBudget = 30 * 1024;
    const int st = env_int("NNVISR_T2F_STAGES", 0);
    if (bits == 8) {
        if (dtype == kF16) return launch_tma(t2f_yuv_tma<FAMILY, uint8_t, __half, float>, a, V, 2, kBudget, st, s);
        return launch_tma(t2f_yuv_tma<FAMILY, uint8_t, float, float>, a, V, 4, kBudget, st, s);
    }
    if (bits == 10) {
        if (dtype == kF16) return launch_tma(t2f_yuv_tma<FAMILY, uint16_t, __half, float>, a, V, 2, kBudget, st, s);
        return launch_tma(t2f_yuv_tma<FAMILY, uint16_t, float, float>, a, V, 4, kBudget, st, s);
    }
    if (dtype == kF16) return launch_tma(t2f_yuv_tma<FAMILY, uint16_t, __half, double>, a, V, 2, kBudget, st, s);
    return launch_tma(t2f_yuv_tma<FAMILY, uint16_t, float, double>, a, V, 4, kBudget, st, s);
}

}  // namespace

cudaError_t launch_f2t_yuv_tma(int family, int bits, int dtype, const F2TArgs &a, cudaStream_t s)
{
    if (family == kYUV420) return f2t_tma_dispatch<kYUV420, true>(bits, dtype, a, s);
    return f2t_tma_dispatch<kYUV444, true>(bits, dtype, a, s);
}

cudaError_t launch_t2f_yuv_tma(int family, int bits, int dtype, const T2FArgs &a, cudaStream_t s)
{
    if (family == kYUV420) return t2f_yuv_tma_dispatch<kYUV420>(bits, dtype, a, s);
    return t2f_yuv_tma_dispatch<kYUV444>(bits, dtype, a, s);
}

cudaError_t launch_f2t_tma(int family, int bits, int dtype, const F2TArgs &a, cudaStream_t s)
{
    switch (family) {
    case kYUV420: return f2t_tma_dispatch<kYUV420>(bits, dtype, a, s);
    case kYUV444: return f2t_tma_dispatch<kYUV444>(bits, dtype, a, s);
    default: return f2t_tma_dispatch<kRGB>(bits, dtype, a, s);
    }
}

cudaError_t launch_t2f_tma(int family, int bits, int dtype, const T2FArgs &a, cudaStream_t s)
{
    switch (family) {
    case kYUV420: return t2f_tma_dispatch<kYUV420>(bits, dtype, a, s);
    case kYUV444: return t2f_tma_dispatch<kYUV444>(bits, dtype, a, s);
    default: return t2f_tma_dispatch<kRGB>(bits, dtype, a, s);
    }
}

}  // namespace nnvisr
