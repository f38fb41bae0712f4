// nnvisr.cpp -- the C ABI (include/nnvisr.h): validation, the host tuple
// planner, scratch management and kernel dispatch.
//
// Citations: PAPER.md = /root/reference/PAPER.md (arXiv 2308.03121); readings
// A1..A16 are listed in DESIGN.md §3.
#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges for nsys / ncu --nvtx
#include "nnvisr.h"

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

using namespace nnvisr;

namespace {

// Scoped NVTX range around each host entry point that plans or launches.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

thread_local std::string g_error;
std::atomic<int64_t> g_launches{0};

nnvisr_status fail(nnvisr_status s, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
nnvisr_status fail(nnvisr_status s, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_error = buf;
    return s;
}

}  // namespace

nnvisr_status nnvisr::set_error(nnvisr_status s, const char *msg)
{
    g_error = msg ? msg : "";
    return s;
}

namespace {

nnvisr_status cuda_fail(cudaError_t e, const char *what)
{
    return fail(NNVISR_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }
int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// A1: ITU matrix coefficients (Kr, Kb).
void kr_kb(int matrix, double &kr, double &kb)
{
    switch (matrix) {
    case NNVISR_BT601: kr = 0.299; kb = 0.114; break;
    case NNVISR_BT709: kr = 0.2126; kb = 0.0722; break;
    default: kr = 0.2627; kb = 0.0593; break;
    }
}

// A pinned-host + device upload slot.  Tables a launch reads (job -> frame
// index, output frame descriptors) are copied host->pinned->device on the
// caller's stream; the slot's event, recorded after the consuming kernels,
// guards reuse.
struct UploadSlot {
    void *host = nullptr;
    void *dev = nullptr;
    cudaEvent_t done = nullptr;
    bool pending = false;
    bool captured = false;  // owned by a CUDA graph capture (never recycled)
};
constexpr size_t kSlotBytes = size_t(1) << 20;
constexpr int kSlots = 8;

}  // namespace

// Called right before each kernel launch.  The launch reports its own errors
// through cudaGetLastError(), so a stale, non-sticky error left by an earlier
// failed runtime call (returned to its caller already) is dropped here
// rather than pinned on this launch.
void nnvisr::count_launch()
{
    g_launches.fetch_add(1, std::memory_order_relaxed);
    (void)cudaGetLastError();
}

struct nnvisr_handle {
    nnvisr_clip_format fmt{};
    nnvisr_network net{};
    int N = 0, M = 0, n = 0, L = 0;
    bool paper = false;  // paper grouping (vs sliding window)
    bool yuv_in = false, yuv_out = false;  // YUV-native network tensors (NEXT-3)
    bool left = false;                      // LEFT (MPEG-2) 4:2:0 siting
    int64_t Hp = 0, Wp = 0, Wo = 0, Ho = 0;
    int64_t Hc = 0, Wc = 0;                 // input chroma tensor plane (YUV input)
    int elem = 4;
    F2TColour f2c{};
    T2FColour t2c{};
    // device state (created on the first device call)
    int device = -1;
    UploadSlot slots[kSlots];
    int next_slot = 0;
    std::vector<std::unique_ptr<UploadSlot>> captured;  // slots of calls recorded into CUDA graphs
    DevFrame *frames = nullptr;
    int64_t frames_cap = 0, frames_base = 0, frames_count = 0;
    bool frames_vec = false;
    int64_t frames_pitch_y = 0, frames_pitch_c = 0;  // uniform pitches of the bound frames, 0 if they differ
    std::vector<nnvisr_frame> frames_host;            // host copy of the bound descriptors
    // host-buffer calls (nnvisr_*_host): device staging rings and copy streams
    struct Stage {
        void *data = nullptr;       // packed frames
        DevFrame *table = nullptr;  // device descriptors of the staged frames
        std::vector<nnvisr_frame> desc;
        int64_t cap = 0;
        cudaEvent_t free_ev = nullptr, ready_ev = nullptr;
        bool used = false;
    };
    Stage in_stage[2], out_stage[2];
    int in_next = 0, out_next = 0;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t d2h_last = nullptr;
    bool d2h_any = false;
    bool force_generic = false;  // NNVISR_FORCE_GENERIC=1: never take the TMA path (tests)
};

namespace {

// --------------------------------------------------------------- planning
// Steps A1-A2 (§3.3; readings A8, A9).  One closed form
// covers both tuple shapes: per scene [s, e) with m = e - s frames, runs
// k = 0 .. ceil(m/n)-1 have
//   base  = min(s + k n, max(s, e - n))          (recycle the last group)
//   in[j] = clamp(base - L + j, s, e - 1)         (duplicate at scene edges)
//   fresh = [s + k n, min(s + (k+1) n, e))
struct PlanSink {
    int64_t *inputs, *fresh;
    int64_t cap, count = 0;
    int N;
    void emit(const int64_t *in, int64_t lo, int64_t hi)
    {
        if (count < cap) {
            std::memcpy(inputs + count * N, in, sizeof(int64_t) * N);
            fresh[2 * count] = lo;
            fresh[2 * count + 1] = hi;
        }
        ++count;
    }
};

void plan_scene(const nnvisr_handle *h, int64_t s, int64_t e, int64_t fresh_begin,
                int64_t fresh_end, PlanSink &out)
{
    const int64_t n = h->n, m = e - s, K = (m + n - 1) / n;
    int64_t in[16];
    for (int64_t k = 0; k < K; ++k) {
        const int64_t lo = s + k * n, hi = std::min(s + (k + 1) * n, e);
        if (lo < fresh_begin || lo >= fresh_end) continue;
        const int64_t base = std::min(s + k * n, std::max(s, e - n));
        for (int j = 0; j < h->N; ++j) in[j] = std::min(std::max(base - h->L + j, s), e - 1);
        out.emit(in, lo, hi);
    }
}

}  // namespace

extern "C" {

const char *nnvisr_last_error(void) { return g_error.c_str(); }
const char *nnvisr_version(void) { return "nnvisr-b200 0.1 (sm_100a)"; }
int64_t nnvisr_launch_count(void) { return g_launches.load(); }

nnvisr_status nnvisr_open(const nnvisr_clip_format *fmt, const nnvisr_network *net, nnvisr_handle **out)
{
    g_error.clear();
    if (!fmt || !net || !out) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    const nnvisr_clip_format f = *fmt;
    const nnvisr_network w = *net;
    if (f.width < 1 || f.height < 1 || f.width > 32768 || f.height > 32768)
        return fail(NNVISR_ERR_INVALID_CONFIG, "frame size %dx%d outside [1, 32768]", f.width, f.height);
    if (f.family != NNVISR_YUV420 && f.family != NNVISR_YUV444 && f.family != NNVISR_RGB)
        return fail(NNVISR_ERR_INVALID_CONFIG, "unknown pixel family %d", f.family);
    if (f.bits != 8 && f.bits != 10 && f.bits != 16)
        return fail(NNVISR_ERR_INVALID_CONFIG, "bits must be 8, 10 or 16 (got %d)", f.bits);
    if (f.family != NNVISR_RGB && (f.matrix < NNVISR_BT601 || f.matrix > NNVISR_BT2020))
        return fail(NNVISR_ERR_INVALID_CONFIG, "unknown colour matrix %d", f.matrix);
    if (f.range != NNVISR_LIMITED && f.range != NNVISR_FULL)
        return fail(NNVISR_ERR_INVALID_CONFIG, "unknown range %d", f.range);
    if (f.chroma_loc != NNVISR_CHROMA_CENTER && f.chroma_loc != NNVISR_CHROMA_LEFT)
        return fail(NNVISR_ERR_INVALID_CONFIG, "unknown chroma siting %d", f.chroma_loc);
    if (f.family == NNVISR_YUV420 && ((f.width | f.height) & 1))
        return fail(NNVISR_ERR_INVALID_CONFIG, "4:2:0 needs even width and height (got %dx%d)", f.width, f.height);

    if (w.input_count < 1 || w.input_count > 16)
        return fail(NNVISR_ERR_INVALID_CONFIG, "input_count must be in [1, 16] (got %d)", w.input_count);
    if (w.output_count < 1 || w.output_count > 16)
        return fail(NNVISR_ERR_INVALID_CONFIG, "output_count must be in [1, 16] (got %d)", w.output_count);
    if (w.n < 1) return fail(NNVISR_ERR_INVALID_CONFIG, "n must be >= 1 (got %d)", w.n);
    if (w.flags & ~31u) return fail(NNVISR_ERR_INVALID_CONFIG, "unknown flag bits 0x%x", w.flags);
    if ((w.flags & (NNVISR_YUV_INPUT | NNVISR_YUV_OUTPUT)) && f.family == NNVISR_RGB)
        return fail(NNVISR_ERR_INVALID_CONFIG, "YUV network tensors need a YUV clip");
    const bool interp = w.flags & NNVISR_INTERPOLATION, extra = w.flags & NNVISR_EXTRA_FRAME,
               dbl = w.flags & NNVISR_DOUBLE_FRAME;
    if (dbl && !interp) return fail(NNVISR_ERR_INVALID_CONFIG, "DOUBLE_FRAME requires INTERPOLATION");
    if (w.sx_num < 1 || w.sx_den < 1 || w.sy_num < 1 || w.sy_den < 1)
        return fail(NNVISR_ERR_INVALID_CONFIG, "scale factor terms must be positive");
    if (interp && !dbl && (w.sx_num != w.sx_den || w.sy_num != w.sy_den))
        return fail(NNVISR_ERR_INVALID_CONFIG, "INTERPOLATION without DOUBLE_FRAME passes input frames through: scale must be 1");
    if ((int64_t)f.width * w.sx_num % w.sx_den || (int64_t)f.height * w.sy_num % w.sy_den)
        return fail(NNVISR_ERR_INVALID_CONFIG, "output size W*sx x H*sy is not integral");
    const int64_t Wo = (int64_t)f.width * w.sx_num / w.sx_den, Ho = (int64_t)f.height * w.sy_num / w.sy_den;
    if (Wo > 65536 || Ho > 65536) return fail(NNVISR_ERR_INVALID_CONFIG, "output size too large");
    if (f.family == NNVISR_YUV420 && ((Wo | Ho) & 1))
        return fail(NNVISR_ERR_INVALID_CONFIG, "4:2:0 output size must be even");
    if (!is_pow2(w.align) || w.align > 256)
        return fail(NNVISR_ERR_INVALID_CONFIG, "align must be a power of two in [1, 256] (got %d)", w.align);
    if (w.dtype != NNVISR_F32 && w.dtype != NNVISR_F16)
        return fail(NNVISR_ERR_INVALID_CONFIG, "unknown tensor dtype %d", w.dtype);

    // tuple shape: paper grouping or sliding window (reading A8)
    const int N = w.input_count, M = w.output_count, n = w.n;
    bool paper = false;
    int L = 0;
    if ((w.left_context == 0 || w.left_context == -1) && N == n + (extra ? 1 : 0)) {
        const bool m_ok = dbl ? (M == 2 * n || M == 2 * n + 1) : (M == n);
        if (!m_ok)
            return fail(NNVISR_ERR_INVALID_CONFIG, "paper grouping: output_count must be %s (got %d)",
                        dbl ? "2n or 2n+1" : "n", M);
        paper = true;
        L = 0;
    } else if ((w.flags & 7u) == 0 && n == 1 && M == 1) {
        L = w.left_context == -1 ? (N - 1) / 2 : w.left_context;
        if (L < 0 || L >= N)
            return fail(NNVISR_ERR_INVALID_CONFIG, "left_context must be in [0, input_count) (got %d)", L);
    } else {
        return fail(NNVISR_ERR_INVALID_CONFIG,
                    "tuple shape: need input_count = n + EXTRA (paper grouping) or flags = 0, n = 1, "
                    "output_count = 1 (sliding window)");
    }

    nnvisr_handle *h = new (std::nothrow) nnvisr_handle();
    if (!h) return fail(NNVISR_ERR_OUT_OF_MEMORY, "handle allocation failed");
    h->fmt = f;
    h->net = w;
    h->N = N; h->M = M; h->n = n; h->L = L; h->paper = paper;
    h->Hp = round_up(f.height, w.align);
    h->Wp = round_up(f.width, w.align);
    h->Wo = Wo; h->Ho = Ho;
    h->elem = w.dtype == NNVISR_F16 ? 2 : 4;
    h->yuv_in = w.flags & NNVISR_YUV_INPUT;
    h->yuv_out = w.flags & NNVISR_YUV_OUTPUT;
    h->left = f.chroma_loc == NNVISR_CHROMA_LEFT;
    h->Hc = f.family == NNVISR_YUV420 ? h->Hp / 2 : h->Hp;
    h->Wc = f.family == NNVISR_YUV420 ? h->Wp / 2 : h->Wp;
    const char *fg = std::getenv("NNVISR_FORCE_GENERIC");
    h->force_generic = fg && fg[0] == '1';

    // A5 dequantisation on 16x codes: luma v = (16c - y_off) * y_scale,
    // chroma P = (s - c_off) * c_scale with s = 16 x (upsampled) code.
    const double k = std::ldexp(1.0, f.bits - 8), full = std::ldexp(1.0, f.bits) - 1.0;
    if (f.range == NNVISR_LIMITED) {
        h->f2c.y_off = (int32_t)(256 * k);
        h->f2c.y_scale = (float)(1.0 / (16.0 * 219.0 * k));
        h->f2c.c_off = (int32_t)(2048 * k);
        h->f2c.c_scale = (float)(1.0 / (16.0 * 224.0 * k));
        h->f2c.u_off = (int32_t)(256 * k);  // c_off - 16*224k/2
    } else {
        h->f2c.y_off = 0;
        h->f2c.y_scale = (float)(1.0 / (16.0 * full));
        h->f2c.c_off = (int32_t)(16 * std::ldexp(1.0, f.bits - 1));
        h->f2c.c_scale = (float)(1.0 / (16.0 * full));
        h->f2c.u_off = 8;  // 16*2^(d-1) - 16*(2^d-1)/2
    }
    // A6 inverse matrix; G in difference form (gray axis exact, reading A16)
    double kr = 0, kb = 0;
    kr_kb(f.matrix, kr, kb);
    const double kg = 1.0 - kr - kb;
    h->f2c.r_pr = (float)(2.0 * (1.0 - kr));
    h->f2c.b_pb = (float)(2.0 * (1.0 - kb));
    h->f2c.g_pb = (float)(kb * 2.0 * (1.0 - kb) / kg);
    h->f2c.g_pr = (float)(kr * 2.0 * (1.0 - kr) / kg);
    h->f2c.y_scale_d = f.range == NNVISR_LIMITED ? 1.0 / (16.0 * 219.0 * k) : 1.0 / (16.0 * full);
    h->f2c.c_scale_d = f.range == NNVISR_LIMITED ? 1.0 / (16.0 * 224.0 * k) : 1.0 / (16.0 * full);
    h->f2c.r_pr_d = 2.0 * (1.0 - kr);
    h->f2c.b_pb_d = 2.0 * (1.0 - kb);
    h->f2c.g_pb_d = kb * 2.0 * (1.0 - kb) / kg;
    h->f2c.g_pr_d = kr * 2.0 * (1.0 - kr) / kg;
    // chroma scale folded into the matrix (common.cuh f2t_colour), rounded once
    h->f2c.r_v = (float)(h->f2c.r_pr_d * h->f2c.c_scale_d);
    h->f2c.b_u = (float)(h->f2c.b_pb_d * h->f2c.c_scale_d);
    h->f2c.g_u = (float)(h->f2c.g_pb_d * h->f2c.c_scale_d);
    h->f2c.g_v = (float)(h->f2c.g_pr_d * h->f2c.c_scale_d);
    // B2/B4 constants
    T2FColour &c = h->t2c;
    c.kr = kr; c.kb = kb; c.db = 2.0 * (1.0 - kb); c.dr = 2.0 * (1.0 - kr);
    c.idb = 1.0 / c.db; c.idr = 1.0 / c.dr;
    if (f.range == NNVISR_LIMITED) { c.ys = 219.0 * k; c.yo = 16.0 * k; c.cs = 224.0 * k; c.co = 128.0 * k; }
    else { c.ys = full; c.yo = 0.0; c.cs = full; c.co = std::ldexp(1.0, f.bits - 1); }
    c.maxc = full;
    c.fkr = (float)c.kr; c.fkb = (float)c.kb; c.fdb = (float)c.db; c.fdr = (float)c.dr;
    c.fidb = 1.0f / c.fdb; c.fidr = 1.0f / c.fdr;
    c.fys_n = (float)(c.ys / full); c.fyo_n = (float)(c.yo / full); c.fcs_n = (float)(c.cs / full);
    c.fco_n = (float)(c.co / full); c.fmaxc = (float)full;
    c.co2 = c.co - 0.5 * c.cs;
    *out = h;
    return NNVISR_OK;
}

nnvisr_status nnvisr_close(nnvisr_handle *h)
{
    g_error.clear();
    if (!h) return NNVISR_OK;
    if (h->device >= 0) {
        int prev = -1;
        cudaGetDevice(&prev);
        if (prev != h->device) cudaSetDevice(h->device);
        for (auto &s : h->slots) {
            if (s.done) { cudaEventSynchronize(s.done); cudaEventDestroy(s.done); }
            if (s.host) cudaFreeHost(s.host);
            if (s.dev) cudaFree(s.dev);
        }
        if (!h->captured.empty()) cudaDeviceSynchronize();  // replays of captured graphs may still read them
        for (auto &s : h->captured) {
            if (s->host) cudaFreeHost(s->host);
            if (s->dev) cudaFree(s->dev);
        }
        if (h->frames) cudaFree(h->frames);
        if (h->h2d) cudaStreamSynchronize(h->h2d);
        if (h->d2h) cudaStreamSynchronize(h->d2h);
        for (auto *ring : {h->in_stage, h->out_stage})
            for (int i = 0; i < 2; ++i) {
                auto &g = ring[i];
                if (g.data) cudaFree(g.data);
                if (g.table) cudaFree(g.table);
                if (g.free_ev) cudaEventDestroy(g.free_ev);
                if (g.ready_ev) cudaEventDestroy(g.ready_ev);
            }
        if (h->h2d) cudaStreamDestroy(h->h2d);
        if (h->d2h) cudaStreamDestroy(h->d2h);
        if (h->d2h_last) cudaEventDestroy(h->d2h_last);
        if (prev >= 0 && prev != h->device) cudaSetDevice(prev);
    }
    delete h;
    return NNVISR_OK;
}

nnvisr_status nnvisr_tensor_shapes(const nnvisr_handle *h, int64_t in_nchw[4], int64_t out_nchw[4])
{
    g_error.clear();
    if (!h) return fail(NNVISR_ERR_INVALID_ARG, "null handle");
    if (in_nchw) { in_nchw[0] = 1; in_nchw[1] = (h->yuv_in ? 1 : 3) * h->N; in_nchw[2] = h->Hp; in_nchw[3] = h->Wp; }
    if (out_nchw) { out_nchw[0] = 1; out_nchw[1] = (h->yuv_out ? 1 : 3) * h->M; out_nchw[2] = h->Ho; out_nchw[3] = h->Wo; }
    return NNVISR_OK;
}

nnvisr_status nnvisr_chroma_shapes(const nnvisr_handle *h, int64_t in_nchw[4], int64_t out_nchw[4])
{
    g_error.clear();
    if (!h) return fail(NNVISR_ERR_INVALID_ARG, "null handle");
    const bool sub = h->fmt.family == NNVISR_YUV420;
    if (in_nchw) {
        in_nchw[0] = h->yuv_in; in_nchw[1] = h->yuv_in ? 2 * h->N : 0;
        in_nchw[2] = h->yuv_in ? h->Hc : 0; in_nchw[3] = h->yuv_in ? h->Wc : 0;
    }
    if (out_nchw) {
        out_nchw[0] = h->yuv_out; out_nchw[1] = h->yuv_out ? 2 * h->M : 0;
        out_nchw[2] = h->yuv_out ? (sub ? h->Ho / 2 : h->Ho) : 0;
        out_nchw[3] = h->yuv_out ? (sub ? h->Wo / 2 : h->Wo) : 0;
    }
    return NNVISR_OK;
}

nnvisr_status nnvisr_plan(const nnvisr_handle *h, int64_t num_frames, const uint8_t *cut,
                          int64_t *run_inputs, int64_t *run_fresh, int64_t cap, int64_t *num_runs)
{
    NvtxRange nvtx_("nnvisr_plan");
    g_error.clear();
    if (!h || !num_runs) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (num_frames < 0) return fail(NNVISR_ERR_INVALID_ARG, "num_frames < 0");
    if (num_frames > 0 && !cut) return fail(NNVISR_ERR_INVALID_ARG, "null cut array");
    if (cap > 0 && (!run_inputs || !run_fresh)) return fail(NNVISR_ERR_INVALID_ARG, "null output arrays");
    PlanSink sink{run_inputs, run_fresh, std::max<int64_t>(cap, 0), 0, h->N};
    int64_t s = 0;
    for (int64_t k = 1; k <= num_frames; ++k) {
        if (k == num_frames || cut[k]) {
            plan_scene(h, s, k, 0, num_frames, sink);
            s = k;
        }
    }
    *num_runs = sink.count;
    if (sink.count > cap) return fail(NNVISR_ERR_CAPACITY, "plan needs %lld runs, capacity %lld",
                                      (long long)sink.count, (long long)cap);
    return NNVISR_OK;
}

nnvisr_status nnvisr_plan_range(const nnvisr_handle *h, int64_t num_frames, int64_t first, int64_t count,
                                const uint8_t *cut, int64_t fresh_begin, int64_t fresh_end,
                                int64_t *run_inputs, int64_t *run_fresh, int64_t cap, int64_t *num_runs)
{
    NvtxRange nvtx_("nnvisr_plan_range");
    g_error.clear();
    if (!h || !num_runs) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (num_frames < 0 || first < 0 || count < 0 || first + count > num_frames)
        return fail(NNVISR_ERR_INVALID_ARG, "window [%lld, %lld) outside the clip of %lld frames",
                    (long long)first, (long long)(first + count), (long long)num_frames);
    if (fresh_begin < 0 || fresh_end > num_frames || fresh_begin > fresh_end)
        return fail(NNVISR_ERR_INVALID_ARG, "bad fresh range [%lld, %lld)", (long long)fresh_begin,
                    (long long)fresh_end);
    if (count > 0 && !cut) return fail(NNVISR_ERR_INVALID_ARG, "null cut array");
    if (cap > 0 && (!run_inputs || !run_fresh)) return fail(NNVISR_ERR_INVALID_ARG, "null output arrays");
    PlanSink sink{run_inputs, run_fresh, std::max<int64_t>(cap, 0), 0, h->N};
    if (fresh_begin == fresh_end) { *num_runs = 0; return NNVISR_OK; }
    if (h->paper && h->n > 1) {
        // a run's phase depends on its scene start, possibly far outside a
        // shard window (SURVEY.md §8(e) "Limitation")
        if (first != 0 || count != num_frames)
            return fail(NNVISR_ERR_UNSUPPORTED, "n > 1 grouping needs the whole clip's cut flags");
        int64_t s = 0;
        for (int64_t k = 1; k <= num_frames; ++k)
            if (k == num_frames || cut[k]) { plan_scene(h, s, k, fresh_begin, fresh_end, sink); s = k; }
    } else {
        const int64_t need_lo = std::max<int64_t>(0, fresh_begin - h->L);
        const int64_t need_hi = std::min<int64_t>(num_frames, fresh_end + h->N - 1 - h->L);
        if (first > need_lo || first + count < need_hi)
            return fail(NNVISR_ERR_INVALID_ARG, "window [%lld, %lld) does not cover [%lld, %lld)",
                        (long long)first, (long long)(first + count), (long long)need_lo, (long long)need_hi);
        // Scene bounds seen from inside the window.  Bounds beyond the window
        // never bind: every clamp argument lies inside the covered range.
        const int64_t end = first + count;
        std::vector<int64_t> scene_end(count);  // first cut after each frame
        int64_t e = end;
        for (int64_t k = end - 1; k >= first; --k) {
            scene_end[k - first] = e;
            if (cut[k - first] && k > 0) e = k;
        }
        int64_t s = first;
        for (int64_t k = first; k < end; ++k) {
            if (k > first && cut[k - first]) s = k;
            if (k < fresh_begin || k >= fresh_end) continue;
            const int64_t ek = scene_end[k - first];
            int64_t in[16];
            for (int j = 0; j < h->N; ++j) in[j] = std::min(std::max(k - h->L + j, s), ek - 1);
            sink.emit(in, k, k + 1);
        }
    }
    *num_runs = sink.count;
    if (sink.count > cap) return fail(NNVISR_ERR_CAPACITY, "plan needs %lld runs, capacity %lld",
                                      (long long)sink.count, (long long)cap);
    return NNVISR_OK;
}

nnvisr_status nnvisr_plan_store(const nnvisr_handle *h, int64_t num_frames, int64_t first, int64_t count,
                                const uint8_t *cut, int64_t fresh_begin, int64_t fresh_end, int64_t *positions,
                                int64_t cap, int64_t *num_positions, int64_t *window_start)
{
    NvtxRange nvtx_("nnvisr_plan_store");
    g_error.clear();
    if (!h || !num_positions) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (h->n != 1) return fail(NNVISR_ERR_UNSUPPORTED, "the padded store needs one fresh frame per tuple (n = 1)");
    if (num_frames < 0 || first < 0 || count < 0 || first + count > num_frames)
        return fail(NNVISR_ERR_INVALID_ARG, "window [%lld, %lld) outside the clip of %lld frames",
                    (long long)first, (long long)(first + count), (long long)num_frames);
    if (fresh_begin < 0 || fresh_end > num_frames || fresh_begin > fresh_end)
        return fail(NNVISR_ERR_INVALID_ARG, "bad fresh range [%lld, %lld)", (long long)fresh_begin,
                    (long long)fresh_end);
    if (count > 0 && !cut) return fail(NNVISR_ERR_INVALID_ARG, "null cut array");
    if (fresh_end > fresh_begin && !window_start) return fail(NNVISR_ERR_INVALID_ARG, "null window_start");
    if (cap > 0 && !positions) return fail(NNVISR_ERR_INVALID_ARG, "null positions");
    const int64_t L = h->L, R = h->N - 1 - h->L;
    const int64_t need_lo = std::max<int64_t>(0, fresh_begin - L);
    const int64_t need_hi = std::min<int64_t>(num_frames, fresh_end + R);
    const int64_t end = first + count;
    if (fresh_end > fresh_begin && (first > need_lo || end < need_hi))
        return fail(NNVISR_ERR_INVALID_ARG, "window [%lld, %lld) does not cover [%lld, %lld)", (long long)first,
                    (long long)end, (long long)need_lo, (long long)need_hi);
    auto cut_at = [&](int64_t k) { return k > 0 && cut[k - first] != 0; };
    // Scenes as seen from the window (bounds beyond it never bind: every
    // clamp argument of an owned tuple lies inside [need_lo, need_hi)).  A
    // scene [s, e) padded with L copies of s and R copies of e-1 holds, at
    // padded index i, frame clamp(s + i - L, s, e - 1), so the window at
    // padded index k - s is tuple k's inputs clamp(k - L + j, s, e - 1)
    // (reading A8 at scene edges).  Only the padded indices the owned tuples
    // read are emitted.
    int64_t P = 0;
    int64_t k = fresh_begin;
    int64_t s = first;
    for (int64_t q = first + 1; q <= k && q < end; ++q)
        if (cut_at(q)) s = q;
    while (k < fresh_end) {
        if (k > fresh_begin && cut_at(k)) s = k;
        int64_t e = k + 1;
        while (e < end && !cut_at(e)) ++e;
        const int64_t b = std::min(e, fresh_end);  // owned fresh frames of this scene: [k, b)
        const int64_t p0 = P;
        for (int64_t i = k - s; i < b - s + h->N - 1; ++i) {
            if (P < cap) positions[P] = std::min(std::max(s + i - L, s), e - 1);
            ++P;
        }
        for (int64_t kk = k; kk < b; ++kk) window_start[kk - fresh_begin] = p0 + (kk - k);
        k = b;
    }
    *num_positions = P;
    if (P > cap) return fail(NNVISR_ERR_CAPACITY, "store layout needs %lld positions, capacity %lld", (long long)P,
                             (long long)cap);
    return NNVISR_OK;
}

nnvisr_status nnvisr_halo_extent(const nnvisr_handle *h, int32_t *left, int32_t *right)
{
    g_error.clear();
    if (!h || !left || !right) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    // inputs of a run: base - L + j (j < N), clamped to its scene; base >= lo
    // - (n-1) (the recycled last run of a scene) and base <= lo
    *left = h->L + (h->paper ? h->n - 1 : 0);
    *right = h->N - 1 - h->L;
    return NNVISR_OK;
}

nnvisr_status nnvisr_plan_range_anchored(const nnvisr_handle *h, int64_t num_frames, int64_t first, int64_t count,
                                         const uint8_t *cut, int64_t scene_start, int64_t fresh_begin,
                                         int64_t fresh_end, int64_t *run_inputs, int64_t *run_fresh, int64_t cap,
                                         int64_t *num_runs)
{
    NvtxRange nvtx_("nnvisr_plan_range_anchored");
    g_error.clear();
    if (!h || !num_runs) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (!h->paper || h->n == 1)  // sliding windows and n = 1: the window alone fixes the plan
        return nnvisr_plan_range(h, num_frames, first, count, cut, fresh_begin, fresh_end, run_inputs, run_fresh,
                                 cap, num_runs);
    if (num_frames < 0 || first < 0 || count < 0 || first + count > num_frames)
        return fail(NNVISR_ERR_INVALID_ARG, "window [%lld, %lld) outside the clip of %lld frames",
                    (long long)first, (long long)(first + count), (long long)num_frames);
    if (fresh_begin < 0 || fresh_end > num_frames || fresh_begin > fresh_end)
        return fail(NNVISR_ERR_INVALID_ARG, "bad fresh range [%lld, %lld)", (long long)fresh_begin,
                    (long long)fresh_end);
    if (count > 0 && !cut) return fail(NNVISR_ERR_INVALID_ARG, "null cut array");
    if (cap > 0 && (!run_inputs || !run_fresh)) return fail(NNVISR_ERR_INVALID_ARG, "null output arrays");
    PlanSink sink{run_inputs, run_fresh, std::max<int64_t>(cap, 0), 0, h->N};
    if (fresh_begin == fresh_end) { *num_runs = 0; return NNVISR_OK; }
    if (scene_start < 0 || scene_start > fresh_begin)
        return fail(NNVISR_ERR_INVALID_ARG, "scene_start %lld outside [0, fresh_begin %lld]", (long long)scene_start,
                    (long long)fresh_begin);
    const int32_t lh = h->L + h->n - 1, rh = h->N - 1 - h->L;
    const int64_t need_lo = std::max<int64_t>(scene_start, fresh_begin - lh);
    const int64_t need_hi = std::min<int64_t>(num_frames, fresh_end + rh);
    const int64_t end = first + count;
    if (first > need_lo || end < need_hi)
        return fail(NNVISR_ERR_INVALID_ARG, "window [%lld, %lld) does not cover [%lld, %lld)", (long long)first,
                    (long long)end, (long long)need_lo, (long long)need_hi);
    auto cut_at = [&](int64_t k) { return k > 0 && cut[k - first] != 0; };
    // the anchor must agree with the window's own flags: no cut in
    // (scene_start, fresh_begin], a cut at scene_start if the window sees it
    for (int64_t k = std::max(scene_start + 1, first); k <= fresh_begin; ++k)
        if (cut_at(k))
            return fail(NNVISR_ERR_INVALID_ARG, "scene_start %lld contradicts the cut at frame %lld",
                        (long long)scene_start, (long long)k);
    if (scene_start > 0 && scene_start >= first && !cut_at(scene_start))
        return fail(NNVISR_ERR_INVALID_ARG, "scene_start %lld is not a cut in the window", (long long)scene_start);
    // Scenes from the anchor on: each ends at the next cut the window shows,
    // else at the window's end, which binds no run whose fresh frame lies in
    // [fresh_begin, fresh_end) (their inputs end before it).  A run's phase is
    // counted from its scene start (§3.3): lo = s + k n.
    const int64_t n = h->n;
    int64_t sc = scene_start;
    while (sc < fresh_end) {
        int64_t e = std::max(sc, fresh_begin) + 1;
        while (e < end && !cut_at(e)) ++e;
        const int64_t m = e - sc, K = (m + n - 1) / n;
        const int64_t k0 = fresh_begin > sc ? (fresh_begin - sc + n - 1) / n : 0;
        int64_t in[16];
        for (int64_t k = k0; k < K; ++k) {
            const int64_t lo = sc + k * n, hi = std::min(sc + (k + 1) * n, e);
            if (lo >= fresh_end) break;
            const int64_t base = std::min(lo, std::max(sc, e - n));
            for (int j = 0; j < h->N; ++j) in[j] = std::min(std::max(base - h->L + j, sc), e - 1);
            sink.emit(in, lo, hi);
        }
        sc = e;
    }
    *num_runs = sink.count;
    if (sink.count > cap) return fail(NNVISR_ERR_CAPACITY, "plan needs %lld runs, capacity %lld",
                                      (long long)sink.count, (long long)cap);
    return NNVISR_OK;
}

}  // extern "C"

// ------------------------------------------------------------ device side
namespace {

nnvisr_status ensure_device(nnvisr_handle *h)
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (h->device < 0) {
        h->device = dev;
        for (auto &s : h->slots) {
            if ((e = cudaHostAlloc(&s.host, kSlotBytes, cudaHostAllocDefault)) != cudaSuccess)
                return cuda_fail(e, "cudaHostAlloc (upload slot)");
            if ((e = cudaMalloc(&s.dev, kSlotBytes)) != cudaSuccess) return cuda_fail(e, "cudaMalloc (upload slot)");
            if ((e = cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming)) != cudaSuccess)
                return cuda_fail(e, "cudaEventCreate");
        }
    } else if (dev != h->device) {
        return fail(NNVISR_ERR_INVALID_ARG, "handle is bound to device %d but device %d is current",
                    h->device, dev);
    }
    return NNVISR_OK;
}

// Take the next upload slot, waiting for its previous consumer if needed.
// On a stream that is being captured into a CUDA graph the call gets a slot
// of its own instead (kept until nnvisr_close): the graph's memcpy node
// re-uploads the same tables, tile counter zeroed, at every replay.
nnvisr_status acquire_slot(nnvisr_handle *h, UploadSlot **out, cudaStream_t st)
{
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaError_t e = cudaStreamIsCapturing(st, &cs);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamIsCapturing");
    if (cs == cudaStreamCaptureStatusActive) {
        auto c = std::make_unique<UploadSlot>();
        c->captured = true;
        cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;  // allocations are allowed here
        cudaThreadExchangeStreamCaptureMode(&mode);
        e = cudaHostAlloc(&c->host, kSlotBytes, cudaHostAllocDefault);
        if (e == cudaSuccess) e = cudaMalloc(&c->dev, kSlotBytes);
        cudaThreadExchangeStreamCaptureMode(&mode);
        if (e != cudaSuccess) {
            if (c->host) cudaFreeHost(c->host);
            return cuda_fail(e, "allocating a capture upload slot");
        }
        *out = c.get();
        h->captured.push_back(std::move(c));
        return NNVISR_OK;
    }
    UploadSlot &s = h->slots[h->next_slot];
    h->next_slot = (h->next_slot + 1) % kSlots;
    if (s.pending) {
        e = cudaEventSynchronize(s.done);
        if (e != cudaSuccess) return cuda_fail(e, "waiting for an upload slot");
        s.pending = false;
    }
    *out = &s;
    return NNVISR_OK;
}

// Append a zeroed 64-bit tile counter (the TMA kernels' dynamic tile
// scheduler) after the `bytes` already staged in the slot; returns its device
// address and grows `bytes`.  It is uploaded with the tables, so every launch
// starts from 0 and the slot's event guards its reuse.
constexpr size_t kCounterBytes = 16;  // alignment slack + the counter
unsigned long long *append_counter(UploadSlot *s, size_t &bytes)
{
    const size_t off = (bytes + 7) & ~size_t(7);
    std::memset(static_cast<char *>(s->host) + off, 0, 8);
    bytes = off + 8;
    return reinterpret_cast<unsigned long long *>(static_cast<char *>(s->dev) + off);
}

nnvisr_status upload(UploadSlot *s, size_t bytes, cudaStream_t st)
{
    cudaError_t e = cudaMemcpyAsync(s->dev, s->host, bytes, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync (upload)");
    return NNVISR_OK;
}

nnvisr_status release_slot(UploadSlot *s, cudaStream_t st)
{
    if (s->captured) return NNVISR_OK;
    cudaError_t e = cudaEventRecord(s->done, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
    s->pending = true;
    return NNVISR_OK;
}

nnvisr_status check_frame(const nnvisr_handle *h, const nnvisr_frame &fr, int64_t w, int64_t hgt,
                          const char *what, int64_t idx, bool *vec)
{
    const int bytes = h->fmt.bits == 8 ? 1 : 2;
    for (int p = 0; p < 3; ++p) {
        const bool sub = h->fmt.family == NNVISR_YUV420 && p > 0;
        const int64_t pw = sub ? w / 2 : w;
        (void)hgt;
        if (!fr.plane[p]) return fail(NNVISR_ERR_INVALID_ARG, "%s %lld: plane %d is null", what, (long long)idx, p);
        if (fr.pitch[p] < pw * bytes || fr.pitch[p] % bytes)
            return fail(NNVISR_ERR_INVALID_ARG, "%s %lld: plane %d pitch %lld invalid (row is %lld bytes)", what,
                        (long long)idx, p, (long long)fr.pitch[p], (long long)(pw * bytes));
        if (reinterpret_cast<uintptr_t>(fr.plane[p]) % bytes)
            return fail(NNVISR_ERR_INVALID_ARG, "%s %lld: plane %d not sample aligned", what, (long long)idx, p);
        if (!aligned16(fr.plane[p]) || fr.pitch[p] % 16) *vec = false;
    }
    return NNVISR_OK;
}

// Uniform plane pitches of a frame list: luma (plane 0) and chroma (planes 1
// and 2, which must agree; for 4:4:4 / RGB also with plane 0), else 0.
void uniform_pitches(const nnvisr_handle *h, const nnvisr_frame *fr, int64_t count, int64_t &py, int64_t &pc)
{
    py = count ? fr[0].pitch[0] : 0;
    pc = count ? fr[0].pitch[1] : 0;
    for (int64_t i = 0; i < count; ++i) {
        if (fr[i].pitch[0] != py) py = 0;
        if (fr[i].pitch[1] != pc || fr[i].pitch[2] != pc) pc = 0;
    }
    if (h->fmt.family != NNVISR_YUV420 && pc != py) py = pc = 0;
}

F2TArgs f2t_args(const nnvisr_handle *h)
{
    F2TArgs a{};
    const int rows = h->fmt.family == NNVISR_YUV420 ? 2 : 1;
    a.W = h->fmt.width; a.H = h->fmt.height; a.Hp = (int32_t)h->Hp; a.Wp = (int32_t)h->Wp;
    a.col_units = (int32_t)((h->Wp + kPx - 1) / kPx);
    a.units = (int32_t)(h->Hp / rows) * a.col_units;
    a.slot_bytes = 3 * h->Hp * h->Wp * h->elem;
    a.vec_out = (h->Wp * h->elem) % 16 == 0;
    a.col = h->f2c;
    a.left = h->left && h->fmt.family == NNVISR_YUV420;
    if (h->yuv_in) {
        a.yuv = 1;
        a.Hc = (int32_t)h->Hc;
        a.Wc = (int32_t)h->Wc;
        a.slot_bytes = h->Hp * h->Wp * h->elem;
        a.slot_bytes2 = 2 * h->Hc * h->Wc * h->elem;
        a.cplane_bytes = h->Hc * h->Wc * h->elem;
    }
    return a;
}

// Destination of an f2t launch.  RGB: dst only.  YUV input: luma at dst, the
// chroma at dst2 (nullptr: the packed tuple layout, chroma right after the
// per_run luma planes of each run), with run strides run_stride / run_stride2.
void set_f2t_dst(const nnvisr_handle *h, F2TArgs &a, char *dst, int64_t run_stride, char *dst2, int64_t run_stride2,
                 int per_run)
{
    a.dst = dst;
    a.run_stride = run_stride;
    if (!h->yuv_in) return;
    if (!dst2) {
        dst2 = dst + per_run * h->Hp * h->Wp * h->elem;
        run_stride2 = run_stride;
    }
    a.dst2 = dst2;
    a.run_stride2 = run_stride2;
    const int64_t al = h->fmt.family == NNVISR_YUV420 ? 4 * h->elem : 16;
    a.vec_out_c = reinterpret_cast<uintptr_t>(dst2) % al == 0 && run_stride2 % al == 0 && a.slot_bytes2 % al == 0 &&
                  a.cplane_bytes % al == 0 && (h->Wc * h->elem) % al == 0;
}

// Bytes of one network input tuple, one store slot, one output tuple.
int64_t in_tuple_bytes(const nnvisr_handle *h)
{
    return h->yuv_in ? h->N * (h->Hp * h->Wp + 2 * h->Hc * h->Wc) * h->elem : 3 * h->N * h->Hp * h->Wp * h->elem;
}
int64_t store_slot_bytes(const nnvisr_handle *h)
{
    return h->yuv_in ? (h->Hp * h->Wp + 2 * h->Hc * h->Wc) * h->elem : 3 * h->Hp * h->Wp * h->elem;
}

nnvisr_status run_f2t(nnvisr_handle *h, F2TArgs a, int64_t jobs, int64_t dests, cudaStream_t st)
{
    a.items = jobs * a.units;
    a.jobs = jobs;
    a.dests = dests;
    // TMA-pipelined path: every copy window 16-byte aligned (planes and
    // pitches 16-byte aligned; windows rounded up into the pitch padding, so
    // any width) and 16-byte tensor rows for the bulk stores
    const int rows = h->fmt.family == NNVISR_YUV420 ? 2 : 1;
    a.rowunits = (int32_t)(h->Hp / rows);
    a.nseg = (int32_t)((h->Wp + kThreads * kPx - 1) / (kThreads * kPx));
    a.tiles = jobs * a.rowunits * a.nseg;
    // YUV-native tensors (NEXT-3): the chroma rows written by bulk stores
    // must be 16-byte aligned too
    const bool yuv_ok = !a.yuv || (reinterpret_cast<uintptr_t>(a.dst2) % 16 == 0 && a.run_stride2 % 16 == 0 &&
                                   a.slot_bytes2 % 16 == 0 && a.cplane_bytes % 16 == 0 &&
                                   (a.Wc * h->elem) % 16 == 0);
    // (the padded width Wp a multiple of 8: whole 8-column groups in the
    // consumers' output staging rows)
    a.tma_ok = !h->force_generic && a.vec_in && a.vec_out && h->Wp % kPx == 0 &&
               reinterpret_cast<uintptr_t>(a.dst) % 16 == 0 && a.run_stride % 16 == 0 && a.slot_bytes % 16 == 0 &&
               yuv_ok;
    cudaError_t e = launch_f2t(h->fmt.family, h->fmt.bits, h->net.dtype, a, st);
    if (e != cudaSuccess) return cuda_fail(e, "f2t kernel launch");
    return NNVISR_OK;
}

// Work list of one f2t launch over `runs` runs of `per_run` slots whose frame
// keys are key[r*per_run + t]: one job per distinct key, with the (run, slot)
// destinations of that key.  Written into `buf` as
// [job_frame: J][job_dst: J+1][dst_code: <= runs*per_run] (int32); returns J.
// Keys < 0 have no destination (nnvisr_frames_to_slots' "leave untouched").
int64_t build_f2t_jobs(const int64_t *key, int64_t runs, int per_run, int64_t key_base, int32_t *buf)
{
    std::vector<std::pair<int64_t, int32_t>> items;
    items.reserve(runs * per_run);
    for (int64_t i = 0; i < runs * per_run; ++i)  // key < 0: no destination
        if (key[i] >= 0) items.push_back({key[i] - key_base, (int32_t)((i / per_run) * 32 + (i % per_run))});
    const int64_t n = (int64_t)items.size();
    std::stable_sort(items.begin(), items.end(),
                     [](const auto &x, const auto &y) { return x.first < y.first; });
    int64_t J = 0;
    for (int64_t i = 0; i < n; ++i)
        if (i == 0 || items[i].first != items[i - 1].first) ++J;
    int32_t *job_frame = buf, *job_dst = buf + J, *dst_code = buf + 2 * J + 1;
    if (J == 0) return 0;
    int64_t j = -1;
    for (int64_t i = 0; i < n; ++i) {
        if (i == 0 || items[i].first != items[i - 1].first) {
            ++j;
            job_frame[j] = (int32_t)items[i].first;
            job_dst[j] = (int32_t)i;
        }
        dst_code[i] = items[i].second;
    }
    job_dst[J] = (int32_t)n;
    return J;
}

T2FArgs t2f_args(const nnvisr_handle *h, int64_t t_h, int64_t t_w)
{
    T2FArgs a{};
    const int rows = h->fmt.family == NNVISR_YUV420 ? 2 : 1;
    a.M = h->M; a.Wo = (int32_t)h->Wo; a.Ho = (int32_t)h->Ho; a.th = t_h; a.tw = t_w;
    a.col_units = (int32_t)((h->Wo + kPx - 1) / kPx);
    a.units = (int32_t)(h->Ho / rows) * a.col_units;
    a.vec_in = (t_w * h->elem) % 16 == 0;
    a.col = h->t2c;
    a.left = h->left && h->fmt.family == NNVISR_YUV420;
    if (h->yuv_out) {
        const bool sub = h->fmt.family == NNVISR_YUV420;
        a.yuv = 1;
        a.thc = sub ? t_h / 2 : t_h;
        a.twc = sub ? t_w / 2 : t_w;
    }
    return a;
}

nnvisr_status run_t2f(nnvisr_handle *h, T2FArgs a, int64_t jobs, cudaStream_t st)
{
    a.items = jobs * a.units;
    const int rows = h->fmt.family == NNVISR_YUV420 ? 2 : 1;
    a.rowunits = (int32_t)(h->Ho / rows);
    a.nseg = (int32_t)((h->Wo + kThreads * kPx - 1) / (kThreads * kPx));
    a.tiles = jobs * a.rowunits * a.nseg;
    // YUV-native tensors (NEXT-3): the chroma rows staged by TMA must be
    // 16-byte aligned too (their base, strides and rows)
    const bool yuv_ok = !a.yuv || (reinterpret_cast<uintptr_t>(a.src2) % 16 == 0 && a.tensor_stride2 % 16 == 0 &&
                                   (a.thc * a.twc * h->elem) % 16 == 0 && (a.twc * h->elem) % 16 == 0);
    // any output width for RGB tensors (a ragged last group stores its valid
    // columns); YUV-native: Wo % 16 (16-byte half-width chroma rows)
    a.tma_ok = !h->force_generic && a.vec_in && a.vec_out && (!a.yuv || h->Wo % 16 == 0) &&
               a.tensor_stride % 16 == 0 &&
               reinterpret_cast<uintptr_t>(a.src) % 16 == 0 && yuv_ok;
    cudaError_t e = launch_t2f(h->fmt.family, h->fmt.bits, h->net.dtype, a, st);
    if (e != cudaSuccess) return cuda_fail(e, "t2f kernel launch");
    return NNVISR_OK;
}

}  // namespace

extern "C" {

nnvisr_status nnvisr_bind_frames(nnvisr_handle *h, int64_t base, const nnvisr_frame *frames, int64_t count)
{
    g_error.clear();
    if (!h) return fail(NNVISR_ERR_INVALID_ARG, "null handle");
    if (count < 0 || (count > 0 && !frames)) return fail(NNVISR_ERR_INVALID_ARG, "bad frame array");
    if (count > INT32_MAX) return fail(NNVISR_ERR_INVALID_ARG, "too many frames");
    bool vec = true;
    for (int64_t i = 0; i < count; ++i) {
        nnvisr_status s = check_frame(h, frames[i], h->fmt.width, h->fmt.height, "frame", base + i, &vec);
        if (s) return s;
    }
    nnvisr_status s = ensure_device(h);
    if (s) return s;
    cudaError_t e;
    // previous batched work may still read the old table
    for (auto &sl : h->slots)
        if (sl.pending && (e = cudaEventSynchronize(sl.done)) != cudaSuccess) return cuda_fail(e, "sync");
    if (count > h->frames_cap) {
        if (h->frames) cudaFree(h->frames);
        h->frames = nullptr;
        h->frames_cap = 0;
        if ((e = cudaMalloc(&h->frames, sizeof(DevFrame) * count)) != cudaSuccess)
            return cuda_fail(e, "cudaMalloc (frame table)");
        h->frames_cap = count;
    }
    static_assert(sizeof(DevFrame) == sizeof(nnvisr_frame), "descriptor layout");
    if (count && (e = cudaMemcpy(h->frames, frames, sizeof(DevFrame) * count, cudaMemcpyHostToDevice)) != cudaSuccess)
        return cuda_fail(e, "cudaMemcpy (frame table)");
    h->frames_base = base;
    h->frames_count = count;
    h->frames_vec = vec;
    uniform_pitches(h, frames, count, h->frames_pitch_y, h->frames_pitch_c);
    h->frames_host.assign(frames, frames + count);
    return NNVISR_OK;
}

nnvisr_status nnvisr_frames_to_tensor(nnvisr_handle *h, const nnvisr_frame *in, void *tensor, void *stream)
{
    NvtxRange nvtx_("nnvisr_frames_to_tensor");
    g_error.clear();
    if (!h || !in || !tensor) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (!aligned16(tensor)) return fail(NNVISR_ERR_INVALID_ARG, "tensor pointer not 16-byte aligned");
    bool vec = true;
    for (int t = 0; t < h->N; ++t) {
        nnvisr_status s = check_frame(h, in[t], h->fmt.width, h->fmt.height, "input slot", t, &vec);
        if (s) return s;
    }
    nnvisr_status s = ensure_device(h);
    if (s) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    UploadSlot *slot = nullptr;
    if ((s = acquire_slot(h, &slot, st))) return s;
    // [DevFrame x N][job_frame, job_dst, dst_code]; identical descriptors are
    // one job (a frame repeated in the tuple is converted once)
    std::vector<int64_t> key(h->N);
    for (int t = 0; t < h->N; ++t) {
        key[t] = t;
        for (int u = 0; u < t; ++u)
            if (!std::memcmp(&in[u], &in[t], sizeof(nnvisr_frame))) { key[t] = u; break; }
    }
    std::memcpy(slot->host, in, sizeof(DevFrame) * h->N);
    int32_t *tab = reinterpret_cast<int32_t *>(static_cast<char *>(slot->host) + sizeof(DevFrame) * h->N);
    const int64_t J = build_f2t_jobs(key.data(), 1, h->N, 0, tab);
    const size_t tab_ints = 2 * J + 1 + h->N;
    size_t bytes = sizeof(DevFrame) * h->N + sizeof(int32_t) * tab_ints;
    unsigned long long *counter = append_counter(slot, bytes);
    if ((s = upload(slot, bytes, st))) return s;
    F2TArgs a = f2t_args(h);
    a.tile_counter = counter;
    const int32_t *dtab = reinterpret_cast<const int32_t *>(static_cast<char *>(slot->dev) + sizeof(DevFrame) * h->N);
    a.frames = static_cast<const DevFrame *>(slot->dev);
    a.job_frame = dtab;
    a.job_dst = dtab + J;
    a.dst_code = dtab + 2 * J + 1;
    set_f2t_dst(h, a, static_cast<char *>(tensor), 0, nullptr, 0, h->N);
    a.vec_in = vec;
    uniform_pitches(h, in, h->N, a.pitch_y, a.pitch_c);
    s = run_f2t(h, a, J, tab[2 * J], st);
    nnvisr_status s2 = release_slot(slot, st);
    return s ? s : s2;
}

// The frames a batched f2t reads: the bound table, or a host-call staging ring.
struct FrameTable {
    const DevFrame *dev;
    int64_t base;
    bool vec;
    int64_t pitch_y, pitch_c;
};

// dst2 / run_stride2: the chroma tensors of a YUV-input network (nullptr:
// packed after the luma of each run, see set_f2t_dst).
static nnvisr_status f2t_indexed_table(nnvisr_handle *h, const FrameTable &tab, const int64_t *frame_idx,
                                       int64_t runs, int per_run, void *dst, int64_t run_stride, cudaStream_t st,
                                       void *dst2 = nullptr, int64_t run_stride2 = 0);

static nnvisr_status f2t_indexed(nnvisr_handle *h, const int64_t *frame_idx, int64_t runs, int per_run,
                                 void *dst, int64_t run_stride, cudaStream_t st, void *dst2 = nullptr,
                                 int64_t run_stride2 = 0)
{
    if (!h->frames) return fail(NNVISR_ERR_INVALID_ARG, "no frames bound (nnvisr_bind_frames)");
    const FrameTable tab{h->frames, h->frames_base, h->frames_vec, h->frames_pitch_y, h->frames_pitch_c};
    return f2t_indexed_table(h, tab, frame_idx, runs, per_run, dst, run_stride, st, dst2, run_stride2);
}

static nnvisr_status f2t_indexed_table(nnvisr_handle *h, const FrameTable &tab, const int64_t *frame_idx,
                                       int64_t runs, int per_run, void *dst, int64_t run_stride, cudaStream_t st,
                                       void *dst2, int64_t run_stride2)
{
    // an upload slot holds 3 ints per (run, slot) plus one; runs per launch
    // are also bounded by the 5-bit slot / run encoding of dst_code
    const int64_t max_runs = std::min<int64_t>((int64_t)((kSlotBytes - kCounterBytes) / sizeof(int32_t) - 1) / (3 * per_run),
                                               (int64_t)(INT32_MAX / 32));
    F2TArgs a = f2t_args(h);
    a.frames = tab.dev;
    a.vec_in = tab.vec;
    a.pitch_y = tab.pitch_y;
    a.pitch_c = tab.pitch_c;
    for (int64_t r0 = 0; r0 < runs; r0 += max_runs) {
        const int64_t nr = std::min(max_runs, runs - r0);
        UploadSlot *slot = nullptr;
        nnvisr_status s = acquire_slot(h, &slot, st);
        if (s) return s;
        int32_t *tbl = static_cast<int32_t *>(slot->host);
        const int64_t J = build_f2t_jobs(frame_idx + r0 * per_run, nr, per_run, tab.base, tbl);
        if (J == 0) {
            release_slot(slot, st);
            continue;
        }
        size_t bytes = sizeof(int32_t) * (2 * J + 1 + nr * per_run);
        a.tile_counter = append_counter(slot, bytes);
        if ((s = upload(slot, bytes, st))) return s;
        const int32_t *dtab = static_cast<const int32_t *>(slot->dev);
        a.job_frame = dtab;
        a.job_dst = dtab + J;
        a.dst_code = dtab + 2 * J + 1;
        set_f2t_dst(h, a, static_cast<char *>(dst) + r0 * run_stride, run_stride,
                    dst2 ? static_cast<char *>(dst2) + r0 * run_stride2 : nullptr, run_stride2, per_run);
        s = run_f2t(h, a, J, tbl[2 * J], st);
        nnvisr_status s2 = release_slot(slot, st);
        if (s) return s;
        if (s2) return s2;
    }
    return NNVISR_OK;
}

nnvisr_status nnvisr_frames_to_tensor_batch(nnvisr_handle *h, const int64_t *run_inputs, int64_t num_runs,
                                            void *tensors, int64_t tensor_stride_bytes, void *stream)
{
    NvtxRange nvtx_("nnvisr_frames_to_tensor_batch");
    g_error.clear();
    if (!h || (num_runs > 0 && (!run_inputs || !tensors))) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (num_runs < 0) return fail(NNVISR_ERR_INVALID_ARG, "num_runs < 0");
    if (num_runs == 0) return NNVISR_OK;
    const int64_t tbytes = in_tuple_bytes(h);
    if (!aligned16(tensors) || tensor_stride_bytes % 16)
        return fail(NNVISR_ERR_INVALID_ARG, "tensors / stride not 16-byte aligned");
    if (num_runs > 1 && tensor_stride_bytes < tbytes)
        return fail(NNVISR_ERR_INVALID_ARG, "tensor stride %lld < tensor size %lld", (long long)tensor_stride_bytes,
                    (long long)tbytes);
    const int64_t jobs = num_runs * h->N;
    for (int64_t j = 0; j < jobs; ++j) {
        const int64_t f = run_inputs[j];
        if (f < h->frames_base || f >= h->frames_base + h->frames_count)
            return fail(NNVISR_ERR_INVALID_ARG, "run %lld slot %lld: frame %lld not bound (bound [%lld, %lld))",
                        (long long)(j / h->N), (long long)(j % h->N), (long long)f, (long long)h->frames_base,
                        (long long)(h->frames_base + h->frames_count));
    }
    nnvisr_status s = ensure_device(h);
    if (s) return s;
    return f2t_indexed(h, run_inputs, num_runs, h->N, tensors, tensor_stride_bytes, static_cast<cudaStream_t>(stream));
}

nnvisr_status nnvisr_frames_to_store(nnvisr_handle *h, int64_t first, int64_t count, void *store, void *stream)
{
    NvtxRange nvtx_("nnvisr_frames_to_store");
    g_error.clear();
    if (!h || (count > 0 && !store)) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (count < 0) return fail(NNVISR_ERR_INVALID_ARG, "count < 0");
    if (count == 0) return NNVISR_OK;
    if (!aligned16(store)) return fail(NNVISR_ERR_INVALID_ARG, "store not 16-byte aligned");
    if (first < h->frames_base || first + count > h->frames_base + h->frames_count)
        return fail(NNVISR_ERR_INVALID_ARG, "frames [%lld, %lld) not bound", (long long)first, (long long)(first + count));
    nnvisr_status s = ensure_device(h);
    if (s) return s;
    std::vector<int64_t> idx(count);
    for (int64_t i = 0; i < count; ++i) idx[i] = first + i;
    return f2t_indexed(h, idx.data(), count, 1, store, store_slot_bytes(h), static_cast<cudaStream_t>(stream));
}

// chroma / stride2: the chroma tensors of a YUV-output network (nullptr: packed
// after the M luma planes of each tuple).
static nnvisr_status t2f_common(nnvisr_handle *h, const void *tensors, int64_t stride, int64_t t_h, int64_t t_w,
                                const nnvisr_frame *out, int64_t count, cudaStream_t st, const void *chroma = nullptr,
                                int64_t stride2 = 0)
{
    if (t_h < h->Ho || t_w < h->Wo)
        return fail(NNVISR_ERR_INVALID_ARG, "tensor %lldx%lld smaller than the output frame %lldx%lld",
                    (long long)t_w, (long long)t_h, (long long)h->Wo, (long long)h->Ho);
    if (!aligned16(tensors) || stride % 16) return fail(NNVISR_ERR_INVALID_ARG, "tensor / stride not 16-byte aligned");
    const bool sub = h->fmt.family == NNVISR_YUV420;
    if (h->yuv_out && sub && ((t_h | t_w) & 1))
        return fail(NNVISR_ERR_INVALID_ARG, "4:2:0 YUV tensors need an even tensor size (got %lldx%lld)",
                    (long long)t_w, (long long)t_h);
    const int64_t lbytes = (h->yuv_out ? 1 : 3) * h->M * t_h * t_w * h->elem;
    const int64_t cplane = h->yuv_out ? (sub ? (t_h / 2) * (t_w / 2) : t_h * t_w) * h->elem : 0;
    const bool packed = h->yuv_out && !chroma;
    if (packed) {
        chroma = static_cast<const char *>(tensors) + lbytes;
        stride2 = stride;
    }
    const int64_t tbytes = packed ? lbytes + 2 * h->M * cplane : lbytes;
    if (count > 1 && stride < tbytes) return fail(NNVISR_ERR_INVALID_ARG, "tensor stride smaller than the tensor");
    if (h->yuv_out && !packed && count > 1 && stride2 < 2 * h->M * cplane)
        return fail(NNVISR_ERR_INVALID_ARG, "chroma stride smaller than the chroma tensor");
    // outputs whose descriptor has plane[0] == NULL are not converted (an
    // output the emission schedule drops, NEXT-1)
    const int64_t all_jobs = count * h->M;
    std::vector<int32_t> codes;
    std::vector<nnvisr_frame> kept;
    bool vec = true, skipped = false;
    for (int64_t j = 0; j < all_jobs; ++j) {
        if (!out[j].plane[0]) {
            skipped = true;
            continue;
        }
        nnvisr_status s = check_frame(h, out[j], h->Wo, h->Ho, "output frame", j, &vec);
        if (s) return s;
    }
    if (skipped) {
        if (count > (INT32_MAX >> 5)) return fail(NNVISR_ERR_INVALID_ARG, "too many tuples");
        for (int64_t j = 0; j < all_jobs; ++j)
            if (out[j].plane[0]) {
                codes.push_back((int32_t)((j / h->M) * 32 + j % h->M));
                kept.push_back(out[j]);
            }
    }
    const int64_t jobs = skipped ? (int64_t)kept.size() : all_jobs;
    const nnvisr_frame *desc = skipped ? kept.data() : out;
    if (jobs == 0) return NNVISR_OK;
    nnvisr_status s = ensure_device(h);
    if (s) return s;
    T2FArgs a = t2f_args(h, t_h, t_w);
    a.tensor_stride = stride;
    a.vec_out = vec;
    if (h->yuv_out) {
        const int64_t al = sub ? 4 * h->elem : 16;
        a.tensor_stride2 = stride2;
        a.vec_in_c = reinterpret_cast<uintptr_t>(chroma) % al == 0 && stride2 % al == 0 && cplane % al == 0 &&
                     (a.twc * h->elem) % al == 0;
    }
    const size_t per_job = sizeof(DevFrame) + (skipped ? sizeof(int32_t) : 0);
    const int64_t per_slot = skipped ? (int64_t)((kSlotBytes - kCounterBytes) / per_job)
                                     : (int64_t)((kSlotBytes - kCounterBytes) / sizeof(DevFrame)) / h->M * h->M;
    for (int64_t j0 = 0; j0 < jobs; j0 += per_slot) {
        const int64_t nj = std::min(per_slot, jobs - j0);
        UploadSlot *slot = nullptr;
        if ((s = acquire_slot(h, &slot, st))) return s;
        std::memcpy(slot->host, desc + j0, sizeof(DevFrame) * nj);
        if (skipped) std::memcpy(static_cast<char *>(slot->host) + sizeof(DevFrame) * nj, codes.data() + j0, sizeof(int32_t) * nj);
        size_t bytes = per_job * nj;
        a.tile_counter = append_counter(slot, bytes);
        if ((s = upload(slot, bytes, st))) return s;
        a.out = static_cast<const DevFrame *>(slot->dev);
        if (skipped) {
            a.job_code = reinterpret_cast<const int32_t *>(static_cast<char *>(slot->dev) + sizeof(DevFrame) * nj);
            a.src = static_cast<const char *>(tensors);  // codes carry absolute tuple indices
            a.src2 = static_cast<const char *>(chroma);
        } else {
            a.job_code = nullptr;
            a.src = static_cast<const char *>(tensors) + (j0 / h->M) * stride;
            a.src2 = chroma ? static_cast<const char *>(chroma) + (j0 / h->M) * stride2 : nullptr;
        }
        s = run_t2f(h, a, nj, st);
        nnvisr_status s2 = release_slot(slot, st);
        if (s) return s;
        if (s2) return s2;
    }
    return NNVISR_OK;
}

nnvisr_status nnvisr_tensor_to_frames(nnvisr_handle *h, const void *tensor, int64_t t_h, int64_t t_w,
                                      const nnvisr_frame *out, void *stream)
{
    NvtxRange nvtx_("nnvisr_tensor_to_frames");
    g_error.clear();
    if (!h || !tensor || !out) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    return t2f_common(h, tensor, 0, t_h, t_w, out, 1, static_cast<cudaStream_t>(stream));
}

nnvisr_status nnvisr_tensor_to_frames_batch(nnvisr_handle *h, const void *tensors, int64_t tensor_stride_bytes,
                                            int64_t t_h, int64_t t_w, const nnvisr_frame *out, int64_t count,
                                            void *stream)
{
    NvtxRange nvtx_("nnvisr_tensor_to_frames_batch");
    g_error.clear();
    if (!h || (count > 0 && (!tensors || !out))) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (count < 0) return fail(NNVISR_ERR_INVALID_ARG, "count < 0");
    if (count == 0) return NNVISR_OK;
    return t2f_common(h, tensors, tensor_stride_bytes, t_h, t_w, out, count, static_cast<cudaStream_t>(stream));
}

nnvisr_status nnvisr_frames_to_tensor_yuv_batch(nnvisr_handle *h, const int64_t *run_inputs, int64_t num_runs,
                                                void *luma, int64_t luma_stride_bytes, void *chroma,
                                                int64_t chroma_stride_bytes, void *stream)
{
    NvtxRange nvtx_("nnvisr_frames_to_tensor_yuv_batch");
    g_error.clear();
    if (!h || (num_runs > 0 && (!run_inputs || !luma || !chroma))) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (!h->yuv_in) return fail(NNVISR_ERR_INVALID_ARG, "the network does not take YUV tensors (NNVISR_YUV_INPUT)");
    if (num_runs < 0) return fail(NNVISR_ERR_INVALID_ARG, "num_runs < 0");
    if (num_runs == 0) return NNVISR_OK;
    if (!aligned16(luma) || luma_stride_bytes % 16)
        return fail(NNVISR_ERR_INVALID_ARG, "luma tensors / stride not 16-byte aligned");
    if (reinterpret_cast<uintptr_t>(chroma) % h->elem || chroma_stride_bytes % h->elem)
        return fail(NNVISR_ERR_INVALID_ARG, "chroma tensors / stride not element aligned");
    if (num_runs > 1 && (luma_stride_bytes < h->N * h->Hp * h->Wp * h->elem ||
                         chroma_stride_bytes < 2 * h->N * h->Hc * h->Wc * h->elem))
        return fail(NNVISR_ERR_INVALID_ARG, "tensor stride smaller than the tensor");
    for (int64_t j = 0; j < num_runs * h->N; ++j)
        if (run_inputs[j] < h->frames_base || run_inputs[j] >= h->frames_base + h->frames_count)
            return fail(NNVISR_ERR_INVALID_ARG, "run %lld: frame %lld not bound", (long long)(j / h->N),
                        (long long)run_inputs[j]);
    nnvisr_status s = ensure_device(h);
    if (s) return s;
    return f2t_indexed(h, run_inputs, num_runs, h->N, luma, luma_stride_bytes, static_cast<cudaStream_t>(stream),
                       chroma, chroma_stride_bytes);
}

nnvisr_status nnvisr_tensor_to_frames_yuv_batch(nnvisr_handle *h, const void *luma, int64_t luma_stride_bytes,
                                                const void *chroma, int64_t chroma_stride_bytes, int64_t t_h,
                                                int64_t t_w, const nnvisr_frame *out, int64_t count, void *stream)
{
    NvtxRange nvtx_("nnvisr_tensor_to_frames_yuv_batch");
    g_error.clear();
    if (!h || (count > 0 && (!luma || !chroma || !out))) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (!h->yuv_out) return fail(NNVISR_ERR_INVALID_ARG, "the network does not produce YUV tensors (NNVISR_YUV_OUTPUT)");
    if (count < 0) return fail(NNVISR_ERR_INVALID_ARG, "count < 0");
    if (count == 0) return NNVISR_OK;
    if (reinterpret_cast<uintptr_t>(chroma) % h->elem || chroma_stride_bytes % h->elem)
        return fail(NNVISR_ERR_INVALID_ARG, "chroma tensors / stride not element aligned");
    return t2f_common(h, luma, luma_stride_bytes, t_h, t_w, out, count, static_cast<cudaStream_t>(stream), chroma,
                      chroma_stride_bytes);
}

nnvisr_status nnvisr_scene_detect(nnvisr_handle *h, int64_t first, int64_t count, double threshold, uint64_t *sad,
                                  uint8_t *cut, void *stream)
{
    NvtxRange nvtx_("nnvisr_scene_detect");
    g_error.clear();
    if (!h || (count > 0 && (!sad || !cut))) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (count < 0 || count > INT32_MAX) return fail(NNVISR_ERR_INVALID_ARG, "bad count");
    if (!(threshold >= 0.0)) return fail(NNVISR_ERR_INVALID_ARG, "threshold must be >= 0");
    if (count == 0) return NNVISR_OK;
    if (!h->frames) return fail(NNVISR_ERR_INVALID_ARG, "no frames bound (nnvisr_bind_frames)");
    if (first < h->frames_base || first + count > h->frames_base + h->frames_count)
        return fail(NNVISR_ERR_INVALID_ARG, "frames [%lld, %lld) not bound", (long long)first, (long long)(first + count));
    nnvisr_status s = ensure_device(h);
    if (s) return s;
    const int vec = h->frames_vec && h->fmt.width % kPx == 0;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    // the kernels read the bound frame table: take an upload slot (no upload)
    // so that its event orders a later nnvisr_bind_frames after them
    UploadSlot *slot = nullptr;
    if ((s = acquire_slot(h, &slot, st))) return s;
    cudaError_t e = launch_scene_detect(h->fmt.family, h->fmt.bits, h->fmt.range, h->fmt.width, h->fmt.height,
                                        h->frames + (first - h->frames_base), (int)count, vec, threshold, sad, cut, st);
    nnvisr_status s2 = release_slot(slot, st);
    if (e != cudaSuccess) return cuda_fail(e, "scene detection launch");
    return s2;
}

int64_t nnvisr_shared_slot_offset(int32_t n, int32_t b, int32_t region, int32_t k, int32_t j)
{
    if (n < 1 || b < 1 || region < 0 || k < 0 || k > n || j < 0 || j >= b) return -1;
    const int64_t base = (int64_t)region * n * b;
    if (k == 0) return base + j;
    if (k == n) return base + 1 + j;
    return base + 1 + b + (int64_t)(k - 1) * b + j;
}

nnvisr_status nnvisr_plan_batches(const nnvisr_handle *h, int64_t num_frames, const uint8_t *cut, int32_t b,
                                  uint8_t *shared, int64_t *lanes, uint8_t *emit, int64_t *slot_frames, int64_t cap,
                                  int64_t *num_batches)
{
    g_error.clear();
    if (!h || !num_batches) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (!h->paper) return fail(NNVISR_ERR_UNSUPPORTED, "batches are planned for the paper's grouping only");
    if (b < 1 || b > 1024) return fail(NNVISR_ERR_INVALID_ARG, "batch size b must be in [1, 1024]");
    if (num_frames < 0 || (num_frames > 0 && !cut)) return fail(NNVISR_ERR_INVALID_ARG, "bad cut array");
    if (cap > 0 && (!shared || !lanes || !emit || !slot_frames))
        return fail(NNVISR_ERR_INVALID_ARG, "null output arrays");
    // the runs of the whole clip, and each scene's run range
    const int N = h->N, n = h->n;
    std::vector<int64_t> ins(std::max<int64_t>(num_frames, 1) * N), fr(std::max<int64_t>(num_frames, 1) * 2);
    PlanSink sink{ins.data(), fr.data(), std::max<int64_t>(num_frames, 1), 0, N};
    std::vector<std::pair<int64_t, int64_t>> scene_runs;  // [first run, end run)
    int64_t s0 = 0;
    for (int64_t k = 1; k <= num_frames; ++k) {
        if (k == num_frames || cut[k]) {
            const int64_t r0 = sink.count;
            plan_scene(h, s0, k, 0, num_frames, sink);
            scene_runs.push_back({r0, sink.count});
            s0 = k;
        }
    }
    const bool extra = h->net.flags & NNVISR_EXTRA_FRAME;
    auto consecutive = [&](int64_t r) {
        for (int k2 = 1; k2 < N; ++k2)
            if (ins[r * N + k2] != ins[r * N] + k2) return false;
        return true;
    };
    int64_t nb = 0;
    for (auto [ra, rb] : scene_runs) {
        for (int64_t c = ra; c < rb; c += b) {
            if (nb < cap) {
                bool all_aligned = true, full = true;
                for (int j = 0; j < b; ++j) {
                    const bool real = c + j < rb;
                    const int64_t r = real ? c + j : rb - 1;
                    lanes[nb * b + j] = r;
                    emit[nb * b + j] = real;
                    full = full && real;
                    // padding lanes (!real) never make a shared batch (full is false);
                    // skipping them also keeps r - 1 >= 0
                    all_aligned = all_aligned && (!real || (consecutive(r) && (j == 0 || ins[r * N] == ins[(r - 1) * N] + n)));
                }
                const bool sh = extra && full && all_aligned;
                shared[nb] = sh;
                int64_t *sf = slot_frames + nb * (int64_t)b * N;
                for (int64_t o = 0; o < (int64_t)b * N; ++o) sf[o] = -1;
                if (sh) {
                    const int64_t f0 = ins[c * N];
                    for (int j = 0; j < b; ++j)
                        for (int k2 = 0; k2 <= n; ++k2)
                            sf[nnvisr_shared_slot_offset(n, b, 0, k2, j)] = f0 + (int64_t)j * n + k2;
                } else {
                    for (int k2 = 0; k2 < N; ++k2)
                        for (int j = 0; j < b; ++j) sf[(int64_t)k2 * b + j] = ins[lanes[nb * b + j] * N + k2];
                }
            }
            ++nb;
        }
    }
    *num_batches = nb;
    if (nb > cap) return fail(NNVISR_ERR_CAPACITY, "plan needs %lld batches, capacity %lld", (long long)nb,
                              (long long)cap);
    return NNVISR_OK;
}

nnvisr_status nnvisr_frames_to_slots(nnvisr_handle *h, const int64_t *slot_frames, int64_t count, void *store,
                                     void *stream)
{
    NvtxRange nvtx_("nnvisr_frames_to_slots");
    g_error.clear();
    if (!h || (count > 0 && (!slot_frames || !store))) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (count < 0) return fail(NNVISR_ERR_INVALID_ARG, "count < 0");
    if (count == 0) return NNVISR_OK;
    if (!aligned16(store)) return fail(NNVISR_ERR_INVALID_ARG, "store not 16-byte aligned");
    for (int64_t i = 0; i < count; ++i) {
        const int64_t f = slot_frames[i];
        if (f < 0) continue;
        if (f < h->frames_base || f >= h->frames_base + h->frames_count)
            return fail(NNVISR_ERR_INVALID_ARG, "slot %lld: frame %lld not bound", (long long)i, (long long)f);
    }
    nnvisr_status s = ensure_device(h);
    if (s) return s;
    return f2t_indexed(h, slot_frames, count, 1, store, store_slot_bytes(h), static_cast<cudaStream_t>(stream));
}

nnvisr_status nnvisr_copy_slot(nnvisr_handle *h, void *store, int64_t src, int64_t dst, void *stream)
{
    g_error.clear();
    if (!h || !store) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (src < 0 || dst < 0) return fail(NNVISR_ERR_INVALID_ARG, "negative slot");
    if (src == dst) return NNVISR_OK;
    nnvisr_status s = ensure_device(h);
    if (s) return s;
    const int64_t slot_bytes = store_slot_bytes(h);
    char *base = static_cast<char *>(store);
    cudaError_t e = cudaMemcpyAsync(base + dst * slot_bytes, base + src * slot_bytes, slot_bytes,
                                    cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync (slot copy)");
    return NNVISR_OK;
}

nnvisr_status nnvisr_copy_slots(nnvisr_handle *h, void *store, int64_t src, int64_t dst, int64_t count, void *stream)
{
    g_error.clear();
    if (!h || (count > 0 && !store)) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (src < 0 || dst < 0 || count < 0) return fail(NNVISR_ERR_INVALID_ARG, "negative slot or count");
    if (count == 0 || src == dst) return NNVISR_OK;
    if (src < dst + count && dst < src + count)
        return fail(NNVISR_ERR_INVALID_ARG, "slot ranges [%lld, +%lld) and [%lld, +%lld) overlap", (long long)src,
                    (long long)count, (long long)dst, (long long)count);
    nnvisr_status s = ensure_device(h);
    if (s) return s;
    const int64_t slot_bytes = store_slot_bytes(h);
    char *base = static_cast<char *>(store);
    cudaError_t e = cudaMemcpyAsync(base + dst * slot_bytes, base + src * slot_bytes, count * slot_bytes,
                                    cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync (region advance)");
    return NNVISR_OK;
}

nnvisr_status nnvisr_schedule_outputs(const nnvisr_handle *h, int64_t num_frames, const uint8_t *cut,
                                      int32_t *source, int64_t *present, int64_t *run_first, int64_t cap_entries,
                                      int64_t cap_runs, int64_t *num_entries, int64_t *num_runs)
{
    g_error.clear();
    if (!h || !num_entries || !num_runs) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (num_frames < 0 || (num_frames > 0 && !cut)) return fail(NNVISR_ERR_INVALID_ARG, "bad cut array");
    if ((cap_entries > 0 && (!source || !present)) || (cap_runs >= 0 && !run_first))
        return fail(NNVISR_ERR_INVALID_ARG, "null output arrays");
    const int N = h->N, n = h->n;
    const int64_t R = std::max<int64_t>(num_frames, 1);
    std::vector<int64_t> ins(R * N), fr(R * 2);
    PlanSink sink{ins.data(), fr.data(), R, 0, N};
    int64_t s0 = 0;
    for (int64_t k = 1; k <= num_frames; ++k)
        if (k == num_frames || cut[k]) {
            plan_scene(h, s0, k, 0, num_frames, sink);
            s0 = k;
        }
    const bool interp = h->net.flags & NNVISR_INTERPOLATION, dbl = h->net.flags & NNVISR_DOUBLE_FRAME;
    int64_t e = 0;
    for (int64_t r = 0; r < sink.count; ++r) {
        if (r <= cap_runs) run_first[r] = e;
        for (int64_t p = fr[2 * r]; p < fr[2 * r + 1]; ++p) {
            int q = 0;  // consumed position of fresh frame p (sliding windows: the single output)
            if (h->paper)
                while (q < n - 1 && ins[r * N + q] != p) ++q;
            auto put = [&](int32_t src, int64_t pres) {
                if (e < cap_entries) {
                    source[e] = src;
                    present[e] = pres;
                }
                ++e;
            };
            if (!interp) {
                put(h->paper ? q : 0, p);
            } else if (!dbl) {
                put(-(q + 1), 2 * p);
                put(q, 2 * p + 1);
            } else {
                put(2 * q, 2 * p);
                put(2 * q + 1, 2 * p + 1);
            }
        }
    }
    if (sink.count <= cap_runs) run_first[sink.count] = e;
    *num_entries = e;
    *num_runs = sink.count;
    if (e > cap_entries || sink.count > cap_runs)
        return fail(NNVISR_ERR_CAPACITY, "schedule needs %lld entries / %lld runs", (long long)e, (long long)sink.count);
    return NNVISR_OK;
}

nnvisr_status nnvisr_copy_frames(nnvisr_handle *h, const int64_t *src_frames, const nnvisr_frame *out, int64_t count,
                                 void *stream)
{
    NvtxRange nvtx_("nnvisr_copy_frames");
    g_error.clear();
    if (!h || (count > 0 && (!src_frames || !out))) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (count <= 0) return count < 0 ? fail(NNVISR_ERR_INVALID_ARG, "count < 0") : NNVISR_OK;
    if (!h->frames) return fail(NNVISR_ERR_INVALID_ARG, "no frames bound (nnvisr_bind_frames)");
    bool vec = true;
    for (int64_t i = 0; i < count; ++i) {
        const int64_t f = src_frames[i];
        if (f < h->frames_base || f >= h->frames_base + h->frames_count)
            return fail(NNVISR_ERR_INVALID_ARG, "copy %lld: frame %lld not bound", (long long)i, (long long)f);
        nnvisr_status s = check_frame(h, out[i], h->fmt.width, h->fmt.height, "pass-through frame", i, &vec);
        if (s) return s;
    }
    nnvisr_status s = ensure_device(h);
    if (s) return s;
    std::vector<nnvisr_frame> src(count);
    for (int64_t i = 0; i < count; ++i) src[i] = h->frames_host[src_frames[i] - h->frames_base];
    const int sb = h->fmt.bits == 8 ? 1 : 2;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    for (int64_t i = 0; i < count; ++i) {
        for (int p = 0; p < 3; ++p) {
            const bool sub = h->fmt.family == NNVISR_YUV420 && p > 0;
            const int64_t w = (sub ? h->fmt.width / 2 : h->fmt.width) * sb, rows = sub ? h->fmt.height / 2 : h->fmt.height;
            cudaError_t e = cudaMemcpy2DAsync(out[i].plane[p], out[i].pitch[p], src[i].plane[p], src[i].pitch[p], w,
                                              rows, cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy2DAsync (pass-through)");
        }
    }
    return NNVISR_OK;
}

}  // extern "C"

// ------------------------------------------------------- host-buffer calls
namespace {

// Packed staging layout of one frame (w x hgt, the clip's family and depth):
// planes at 16-byte aligned offsets with 16-byte aligned pitches.
struct PackedLayout {
    int64_t off[3], pitch[3], rows[3], row_bytes[3], frame_bytes;
    PackedLayout(const nnvisr_handle *h, int64_t w, int64_t hgt)
    {
        const int sb = h->fmt.bits == 8 ? 1 : 2;
        int64_t o = 0;
        for (int p = 0; p < 3; ++p) {
            const bool sub = h->fmt.family == NNVISR_YUV420 && p > 0;
            row_bytes[p] = (sub ? w / 2 : w) * sb;
            rows[p] = sub ? hgt / 2 : hgt;
            pitch[p] = round_up(row_bytes[p], 16);
            off[p] = o;
            o = round_up(o + pitch[p] * rows[p], 16);
        }
        frame_bytes = round_up(o, 256);
    }
};

nnvisr_status ensure_streams(nnvisr_handle *h)
{
    cudaError_t e;
    if (!h->h2d && (e = cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking)) != cudaSuccess)
        return cuda_fail(e, "cudaStreamCreate (h2d)");
    if (!h->d2h && (e = cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking)) != cudaSuccess)
        return cuda_fail(e, "cudaStreamCreate (d2h)");
    if (!h->d2h_last && (e = cudaEventCreateWithFlags(&h->d2h_last, cudaEventDisableTiming)) != cudaSuccess)
        return cuda_fail(e, "cudaEventCreate");
    return NNVISR_OK;
}

// Grow a staging slot to `count` frames of layout L (device memory + device
// descriptor table); growing waits for the device to drain.
nnvisr_status ensure_stage(nnvisr_handle::Stage &g, int64_t count, const PackedLayout &L)
{
    cudaError_t e;
    if (!g.free_ev) {
        if ((e = cudaEventCreateWithFlags(&g.free_ev, cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&g.ready_ev, cudaEventDisableTiming)) != cudaSuccess)
            return cuda_fail(e, "cudaEventCreate (stage)");
    }
    if (count > g.cap || (count && g.desc.size() && g.desc[0].pitch[0] != L.pitch[0])) {
        if ((e = cudaDeviceSynchronize()) != cudaSuccess) return cuda_fail(e, "staging resize");
        if (g.data) cudaFree(g.data);
        if (g.table) cudaFree(g.table);
        g.data = nullptr;
        g.table = nullptr;
        g.cap = 0;
        if ((e = cudaMalloc(&g.data, L.frame_bytes * count)) != cudaSuccess) return cuda_fail(e, "cudaMalloc (staging)");
        if ((e = cudaMalloc(&g.table, sizeof(DevFrame) * count)) != cudaSuccess)
            return cuda_fail(e, "cudaMalloc (staging table)");
        g.desc.resize(count);
        for (int64_t i = 0; i < count; ++i)
            for (int p = 0; p < 3; ++p) {
                g.desc[i].plane[p] = static_cast<char *>(g.data) + i * L.frame_bytes + L.off[p];
                g.desc[i].pitch[p] = L.pitch[p];
            }
        if ((e = cudaMemcpy(g.table, g.desc.data(), sizeof(DevFrame) * count, cudaMemcpyHostToDevice)) != cudaSuccess)
            return cuda_fail(e, "cudaMemcpy (staging table)");
        g.cap = count;
    }
    return NNVISR_OK;
}

nnvisr_status copy_frame_planes(const nnvisr_frame &dst, const nnvisr_frame &src, const PackedLayout &L,
                                cudaMemcpyKind kind, cudaStream_t st)
{
    for (int p = 0; p < 3; ++p) {
        cudaError_t e = cudaMemcpy2DAsync(dst.plane[p], dst.pitch[p], src.plane[p], src.pitch[p], L.row_bytes[p],
                                          L.rows[p], kind, st);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy2DAsync (host frames)");
    }
    return NNVISR_OK;
}

// Frames count..: dst[i] <- src[i] (plane[0] == NULL on either side: skipped).
// When the packed layout has no padding at all (pitch = row bytes, planes
// and frames back to back) and consecutive frames sit back to back on both
// sides, a run of them moves as ONE copy (small frames: one call instead of
// three per frame); otherwise plane by plane.
nnvisr_status copy_frames_coalesced(const nnvisr_frame *dst, const nnvisr_frame *src, int64_t count,
                                    const PackedLayout &L, cudaMemcpyKind kind, cudaStream_t st)
{
    bool gapless = L.frame_bytes == L.off[2] + L.pitch[2] * L.rows[2];
    for (int p = 0; p < 3; ++p) {
        gapless = gapless && L.pitch[p] == L.row_bytes[p];
        if (p < 2) gapless = gapless && L.off[p + 1] == L.off[p] + L.pitch[p] * L.rows[p];
    }
    auto at = [&](const nnvisr_frame &f, const char *base) {
        for (int p = 0; p < 3; ++p)
            if (static_cast<const char *>(f.plane[p]) != base + L.off[p] || f.pitch[p] != L.pitch[p]) return false;
        return true;
    };
    for (int64_t i = 0; i < count;) {
        if (!dst[i].plane[0] || !src[i].plane[0]) {
            ++i;
            continue;
        }
        const char *sb = static_cast<const char *>(src[i].plane[0]);
        const char *db = static_cast<const char *>(dst[i].plane[0]);
        int64_t j = i;
        while (gapless && j < count && dst[j].plane[0] && src[j].plane[0] && at(src[j], sb + (j - i) * L.frame_bytes) &&
               at(dst[j], db + (j - i) * L.frame_bytes))
            ++j;
        if (j - i >= 2) {
            cudaError_t e = cudaMemcpyAsync(const_cast<char *>(db), sb, (j - i) * L.frame_bytes, kind, st);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync (host frames)");
            i = j;
            continue;
        }
        nnvisr_status s = copy_frame_planes(dst[i], src[i], L, kind, st);
        if (s) return s;
        ++i;
    }
    return NNVISR_OK;
}

}  // namespace

extern "C" {

nnvisr_status nnvisr_frames_to_tensor_batch_host(nnvisr_handle *h, const nnvisr_frame *host_frames, int64_t base,
                                                 int64_t count, const int64_t *run_inputs, int64_t num_runs,
                                                 void *tensors, int64_t tensor_stride_bytes, void *stream)
{
    NvtxRange nvtx_("nnvisr_frames_to_tensor_batch_host");
    g_error.clear();
    if (!h || (count > 0 && !host_frames) || (num_runs > 0 && (!run_inputs || !tensors)))
        return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (count < 0 || num_runs < 0) return fail(NNVISR_ERR_INVALID_ARG, "negative count");
    if (num_runs == 0) return NNVISR_OK;
    if (!aligned16(tensors) || tensor_stride_bytes % 16)
        return fail(NNVISR_ERR_INVALID_ARG, "tensors / stride not 16-byte aligned");
    const int64_t tbytes = in_tuple_bytes(h);
    if (num_runs > 1 && tensor_stride_bytes < tbytes) return fail(NNVISR_ERR_INVALID_ARG, "tensor stride too small");
    for (int64_t j = 0; j < num_runs * h->N; ++j)
        if (run_inputs[j] < base || run_inputs[j] >= base + count)
            return fail(NNVISR_ERR_INVALID_ARG, "run %lld: frame %lld not among the host frames [%lld, %lld)",
                        (long long)(j / h->N), (long long)run_inputs[j], (long long)base, (long long)(base + count));
    for (int64_t i = 0; i < count; ++i)
        for (int p = 0; p < 3; ++p)
            if (!host_frames[i].plane[p]) return fail(NNVISR_ERR_INVALID_ARG, "host frame %lld: null plane", (long long)i);
    nnvisr_status s = ensure_device(h);
    if (s || (s = ensure_streams(h))) return s;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const PackedLayout L(h, h->fmt.width, h->fmt.height);
    auto &g = h->in_stage[h->in_next];
    h->in_next ^= 1;
    if ((s = ensure_stage(g, count, L))) return s;
    cudaError_t e;
    // the kernels that last read this staging slot must be done before the upload
    if (g.used && (e = cudaStreamWaitEvent(h->h2d, g.free_ev, 0)) != cudaSuccess) return cuda_fail(e, "wait");
    if ((s = copy_frames_coalesced(g.desc.data(), host_frames, count, L, cudaMemcpyHostToDevice, h->h2d))) return s;
    if ((e = cudaEventRecord(g.ready_ev, h->h2d)) != cudaSuccess || (e = cudaStreamWaitEvent(st, g.ready_ev, 0)) != cudaSuccess)
        return cuda_fail(e, "upload event");
    const FrameTable tab{g.table, base, true, L.pitch[0], L.pitch[1]};
    s = f2t_indexed_table(h, tab, run_inputs, num_runs, h->N, tensors, tensor_stride_bytes, st);
    if (s) return s;
    if ((e = cudaEventRecord(g.free_ev, st)) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
    g.used = true;
    return NNVISR_OK;
}

nnvisr_status nnvisr_tensor_to_frames_batch_host(nnvisr_handle *h, const void *tensors, int64_t tensor_stride_bytes,
                                                 int64_t t_h, int64_t t_w, const nnvisr_frame *host_out, int64_t count,
                                                 void *stream)
{
    NvtxRange nvtx_("nnvisr_tensor_to_frames_batch_host");
    g_error.clear();
    if (!h || (count > 0 && (!tensors || !host_out))) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (count < 0) return fail(NNVISR_ERR_INVALID_ARG, "count < 0");
    if (count == 0) return NNVISR_OK;
    nnvisr_status s = ensure_device(h);
    if (s || (s = ensure_streams(h))) return s;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t jobs = count * h->M;
    const PackedLayout L(h, h->Wo, h->Ho);
    auto &g = h->out_stage[h->out_next];
    h->out_next ^= 1;
    if ((s = ensure_stage(g, jobs, L))) return s;
    cudaError_t e;
    // the download that last read this staging slot must be done before t2f rewrites it
    if (g.used && (e = cudaStreamWaitEvent(st, g.free_ev, 0)) != cudaSuccess) return cuda_fail(e, "wait");
    std::vector<nnvisr_frame> dev_out(jobs);
    for (int64_t j = 0; j < jobs; ++j) {
        dev_out[j] = g.desc[j];
        if (!host_out[j].plane[0]) dev_out[j].plane[0] = nullptr;  // output not presented
    }
    if ((s = t2f_common(h, tensors, tensor_stride_bytes, t_h, t_w, dev_out.data(), count, st))) return s;
    if ((e = cudaEventRecord(g.ready_ev, st)) != cudaSuccess || (e = cudaStreamWaitEvent(h->d2h, g.ready_ev, 0)) != cudaSuccess)
        return cuda_fail(e, "download event");
    if ((s = copy_frames_coalesced(host_out, g.desc.data(), jobs, L, cudaMemcpyDeviceToHost, h->d2h))) return s;
    if ((e = cudaEventRecord(g.free_ev, h->d2h)) != cudaSuccess || (e = cudaEventRecord(h->d2h_last, h->d2h)) != cudaSuccess)
        return cuda_fail(e, "cudaEventRecord");
    g.used = true;
    h->d2h_any = true;
    return NNVISR_OK;
}

// ---- peer mapping (multi-GPU halo) ----

static_assert(sizeof(cudaIpcMemHandle_t) == sizeof(((nnvisr_peer_handle *)nullptr)->ipc), "IPC handle size");

nnvisr_status nnvisr_peer_export(const void *dev_ptr, nnvisr_peer_handle *out)
{
    g_error.clear();
    if (!dev_ptr || !out) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    cudaPointerAttributes at{};
    cudaError_t e = cudaPointerGetAttributes(&at, dev_ptr);
    if (e != cudaSuccess) return cuda_fail(e, "cudaPointerGetAttributes");
    if (at.type != cudaMemoryTypeDevice) return fail(NNVISR_ERR_INVALID_ARG, "not a device pointer");
    // IPC exports whole allocations: find the one holding dev_ptr (a caching
    // allocator hands out pointers inside larger cudaMalloc blocks)
    using AddressRange = int (*)(unsigned long long *, size_t *, unsigned long long);
    static AddressRange range = nullptr;
    if (!range) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
            return fail(NNVISR_ERR_CUDA, "cuMemGetAddressRange entry point unavailable");
        range = reinterpret_cast<AddressRange>(fn);
    }
    unsigned long long base = 0;
    size_t size = 0;
    if (range(&base, &size, reinterpret_cast<unsigned long long>(dev_ptr)) != 0)
        return fail(NNVISR_ERR_CUDA, "cuMemGetAddressRange failed");
    cudaIpcMemHandle_t ih;
    e = cudaIpcGetMemHandle(&ih, reinterpret_cast<void *>(base));
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
    std::memcpy(out->ipc, &ih, sizeof ih);
    out->offset = static_cast<int64_t>(reinterpret_cast<unsigned long long>(dev_ptr) - base);
    return NNVISR_OK;
}

namespace {
std::mutex g_peer_mu;
std::map<uintptr_t, void *> g_peer_bases;  // imported pointer -> mapped allocation base
}  // namespace

nnvisr_status nnvisr_peer_import(const nnvisr_peer_handle *in, void **dev_ptr)
{
    g_error.clear();
    if (!in || !dev_ptr) return fail(NNVISR_ERR_INVALID_ARG, "null argument");
    if (in->offset < 0) return fail(NNVISR_ERR_INVALID_ARG, "negative offset");
    cudaIpcMemHandle_t ih;
    std::memcpy(&ih, in->ipc, sizeof ih);
    void *base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, ih, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
    *dev_ptr = static_cast<char *>(base) + in->offset;
    std::lock_guard<std::mutex> lk(g_peer_mu);
    g_peer_bases[reinterpret_cast<uintptr_t>(*dev_ptr)] = base;
    return NNVISR_OK;
}

nnvisr_status nnvisr_peer_close(void *dev_ptr)
{
    g_error.clear();
    void *base = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_peer_mu);
        auto it = g_peer_bases.find(reinterpret_cast<uintptr_t>(dev_ptr));
        if (it == g_peer_bases.end()) return fail(NNVISR_ERR_INVALID_ARG, "pointer was not imported by nnvisr_peer_import");
        base = it->second;
        g_peer_bases.erase(it);
    }
    cudaError_t e = cudaIpcCloseMemHandle(base);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
    return NNVISR_OK;
}

nnvisr_status nnvisr_release_graph_tables(nnvisr_handle *h)
{
    g_error.clear();
    if (!h) return fail(NNVISR_ERR_INVALID_ARG, "null handle");
    if (h->captured.empty()) return NNVISR_OK;
    cudaError_t e = cudaDeviceSynchronize();  // no replay may still read them
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceSynchronize");
    for (auto &c : h->captured) {
        if (c->host) cudaFreeHost(c->host);
        if (c->dev) cudaFree(c->dev);
    }
    h->captured.clear();
    return NNVISR_OK;
}

nnvisr_status nnvisr_host_fence(nnvisr_handle *h, void *stream)
{
    g_error.clear();
    if (!h) return fail(NNVISR_ERR_INVALID_ARG, "null handle");
    if (!h->d2h_any) return NNVISR_OK;
    cudaError_t e = cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), h->d2h_last, 0);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamWaitEvent");
    return NNVISR_OK;
}

}  // extern "C"
