/*
 * nnvisr_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, scalar, double-precision CPU implementation of what the
 * NNVISR frame<->tensor hot path computes (arXiv 2308.03121, §3.1 and
 * §3.3; the silent points follow the readings A1..A22 listed in DESIGN.md §3,
 * which restate SURVEY.md §8(c)).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  The
 * product path (paper_2308_03121_b200/) never links, imports or calls it, and
 * it shares no code, header, table or constant generator with that path.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared (no SIMD intrinsics,
 * no fused multiply-add, so every double operation is the one written here).
 *
 * Every entry point returns 0 on success and a negative number on a bad
 * argument.  All buffers are host memory owned by the caller.
 *
 * Parity status per function (see DESIGN.md §4 "pins"):
 *   oracle_plan            pinned (SPEC examples, brute force, hand lists)
 *   oracle_f2t             pinned (textbook matrices, round trip, chroma ramp)
 *   oracle_t2f             pinned (colour-bar code table, gray axis, round trip)
 *   oracle_half_from_double pinned (numpy float16 RNE conversion)
 *   oracle_f2t_sited / oracle_t2f_sited (LEFT siting) pinned (co-sited linear
 *                          fields, LEFT == 4:4:4 path, down/up identity)
 *   oracle_f2t_yuv / oracle_t2f_yuv pinned (range endpoints, affine shape,
 *                          gray vs RGB path, exact round trip, B4 specials)
 *   oracle_scene_detect    pinned (SPEC scenedetect examples, numpy SAD)
 *   oracle_rgb_to_codes / oracle_codes_to_rgb  pinned (colour-bar table)
 *   chroma siting / padding / channel order / even-N centring: conventions,
 *   "parity unpinned" beyond internal consistency (readings A5-A8).
 */
#include <fenv.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

/* ---- enumerations (numeric values documented in DESIGN.md §2) ---------- */
enum { OR_YUV420 = 0, OR_YUV444 = 1, OR_RGB = 2 };
enum { OR_BT601 = 0, OR_BT709 = 1, OR_BT2020 = 2 };
enum { OR_LIMITED = 0, OR_FULL = 1 };
enum { OR_F32 = 0, OR_F16 = 1 };

typedef struct {
    int32_t width, height;   /* luma samples */
    int32_t family;          /* OR_YUV420 | OR_YUV444 | OR_RGB */
    int32_t bits;            /* 8 | 10 | 16; stored as u8 when bits == 8, else u16 */
    int32_t matrix;          /* OR_BT601 | OR_BT709 | OR_BT2020 */
    int32_t range;           /* OR_LIMITED | OR_FULL */
} oracle_format;

/* ---- A1: matrix coefficients (Kr, Kb) of ITU-R BT.601 / BT.709 / BT.2020
 * (non-constant luminance).  The paper only says the network is chosen per
 * colourspace (§3.1, "same pixel value can and usually mean
 * different colors under different colorspace"); the numbers are the ITU
 * ones SPEC.md lists ([MODULE] colorproc, ColorSpace). */
static int kr_kb(int matrix, double *kr, double *kb)
{
    switch (matrix) {
    case OR_BT601:  *kr = 0.299;  *kb = 0.114;  return 0;
    case OR_BT709:  *kr = 0.2126; *kb = 0.0722; return 0;
    case OR_BT2020: *kr = 0.2627; *kb = 0.0593; return 0;
    default: return -1;
    }
}

/* ---- tuple planning (§3.1 "n", flags; §3.3 grouping rules) ----
 *
 * Scenes: cut[k] != 0 means a scene starts at k (a cut between k-1 and k);
 * cut[0] is ignored and the clip ends act as cuts (reading A9; §3.2
 * "standard way to signal the occurence of scene change").
 *
 * Two tuple shapes (reading A8 / DESIGN.md §3):
 *   paper grouping (left_context == 0 and input_count in {n, n+1}):
 *     PAPER.md §3.3: "NNVISR always grouping frames within a scene ... For
 *     interpolation network, NNVISR duplicates the last frame of the scene.
 *     If the last group doesn't have enough frames for network, last frames
 *     from the previous group is recycled ... If the whole scene does not
 *     contain enough input frames then the last frame is further duplicated"
 *     -- operationalised as SPEC.md [MODULE] grouper, plan_scene.
 *   sliding window (n == 1, any input_count N, left context L < N):
 *     frame t is the fresh frame; the window t-L .. t-L+N-1 never crosses a
 *     scene edge, so positions outside the scene repeat the scene's first or
 *     last frame (the same duplication rule applied at both edges).
 *
 * Output: run_inputs[r*N + j] (absolute frame index), run_fresh[2r], [2r+1]
 * = half-open fresh interval.  Returns the number of runs, or -1 if cap is
 * too small / arguments are invalid.
 */
static int64_t plan_scene_paper(int64_t s, int64_t e, int n, int N,
                                int64_t *run_inputs, int64_t *run_fresh,
                                int64_t cap, int64_t r)
{
    int64_t m = e - s;
    int64_t K = (m + n - 1) / n;              /* runs per scene = ceil(m/n) */
    for (int64_t i = 0; i < K; ++i) {
        int64_t consumed[64];
        int64_t fresh_lo, fresh_hi;
        if (i < K - 1) {
            /* an ordinary group: frames i*n .. i*n+n-1 of the scene */
            for (int j = 0; j < n; ++j) consumed[j] = s + i * n + j;
            fresh_lo = s + i * n;
            fresh_hi = s + (i + 1) * n;
        } else if (m >= n) {
            /* last group short: recycle frames of the previous group so the
             * run consumes the last n frames of the scene */
            for (int j = 0; j < n; ++j) consumed[j] = e - n + j;
            fresh_lo = s + i * n;
            fresh_hi = e;
        } else {
            /* whole scene too short: the last frame is further duplicated */
            for (int j = 0; j < n; ++j) consumed[j] = (j < m) ? s + j : e - 1;
            fresh_lo = s;
            fresh_hi = e;
        }
        if (r >= cap) return -1;
        for (int j = 0; j < n; ++j) run_inputs[r * N + j] = consumed[j];
        if (N == n + 1) {
            /* "Extra frame": the frame after the group, or, at the end of
             * the scene, a duplicate of the scene's last frame */
            int64_t next = consumed[n - 1] + 1;
            if (i == K - 1 || next >= e) next = e - 1;
            run_inputs[r * N + n] = next;
        }
        run_fresh[2 * r] = fresh_lo;
        run_fresh[2 * r + 1] = fresh_hi;
        ++r;
    }
    return r;
}

static int64_t plan_scene_window(int64_t s, int64_t e, int N, int L,
                                 int64_t *run_inputs, int64_t *run_fresh,
                                 int64_t cap, int64_t r)
{
    for (int64_t t = s; t < e; ++t) {
        if (r >= cap) return -1;
        for (int j = 0; j < N; ++j) {
            int64_t f = t - L + j;
            if (f < s) f = s;            /* duplicate the scene's first frame */
            if (f > e - 1) f = e - 1;    /* duplicate the scene's last frame  */
            run_inputs[r * N + j] = f;
        }
        run_fresh[2 * r] = t;
        run_fresh[2 * r + 1] = t + 1;
        ++r;
    }
    return r;
}

int64_t oracle_plan(int64_t num_frames, const uint8_t *cut, int n, int N, int L,
                    int64_t *run_inputs, int64_t *run_fresh, int64_t cap)
{
    if (num_frames < 0 || n < 1 || N < 1 || N > 64 || L < 0 || L >= N) return -1;
    int paper = (L == 0 && (N == n || N == n + 1));
    int window = (n == 1);
    if (!paper && !window) return -1;
    int64_t r = 0, s = 0;
    for (int64_t k = 1; k <= num_frames; ++k) {
        if (k == num_frames || cut[k]) {
            /* scene [s, k) */
            if (paper)
                r = plan_scene_paper(s, k, n, N, run_inputs, run_fresh, cap, r);
            else
                r = plan_scene_window(s, k, N, L, run_inputs, run_fresh, cap, r);
            if (r < 0) return -1;
            s = k;
        }
    }
    return r;
}

/* The sliding-window planner on its own (used for n == 1 windows even when
 * L == 0 and N <= 2, where both readings coincide; tests check they agree). */
int64_t oracle_plan_window(int64_t num_frames, const uint8_t *cut, int N, int L,
                           int64_t *run_inputs, int64_t *run_fresh, int64_t cap)
{
    if (num_frames < 0 || N < 1 || N > 64 || L < 0 || L >= N) return -1;
    int64_t r = 0, s = 0;
    for (int64_t k = 1; k <= num_frames; ++k) {
        if (k == num_frames || cut[k]) {
            r = plan_scene_window(s, k, N, L, run_inputs, run_fresh, cap, r);
            if (r < 0) return -1;
            s = k;
        }
    }
    return r;
}

/* ---- IEEE binary16 rounding (reading A12: round to nearest, ties to even,
 * subnormals kept, overflow to infinity).  Written out from the format
 * definition: 1 sign bit, 5 exponent bits (bias 15), 10 fraction bits. */
uint16_t oracle_half_from_double(double v)
{
    uint16_t sign = signbit(v) ? 0x8000u : 0u;
    if (isnan(v)) return 0x7e00u;
    double a = fabs(v);
    if (isinf(a)) return sign | 0x7c00u;
    if (a == 0.0) return sign;
    int e;
    frexp(a, &e);                 /* a = f * 2^e, f in [0.5, 1) */
    int exp_unbiased = e - 1;     /* a = 1.xxx * 2^(e-1) */
    if (exp_unbiased < -14) exp_unbiased = -14;     /* subnormal spacing */
    double quantum = ldexp(1.0, exp_unbiased - 10); /* spacing of halves here */
    double q = a / quantum;                          /* exact (power of 2) */
    double qi = nearbyint(q);                        /* ties to even */
    /* qi * quantum is the rounded magnitude */
    double rounded = qi * quantum;
    if (rounded > 65504.0) return sign | 0x7c00u;   /* beyond the largest half */
    if (rounded < ldexp(1.0, -14)) {
        /* subnormal: fraction = rounded / 2^-24 */
        uint16_t frac = (uint16_t)(rounded / ldexp(1.0, -24));
        return sign | frac;
    }
    int e2;
    double f2 = frexp(rounded, &e2);  /* rounded = f2 * 2^e2 */
    int biased = (e2 - 1) + 15;
    uint16_t frac = (uint16_t)((f2 * 2.0 - 1.0) * 1024.0);
    return sign | (uint16_t)(biased << 10) | frac;
}

double oracle_double_from_half(uint16_t h)
{
    int sign = (h >> 15) & 1, ex = (h >> 10) & 31, fr = h & 1023;
    double v;
    if (ex == 0) v = ldexp((double)fr, -24);
    else if (ex == 31) v = fr ? NAN : INFINITY;
    else v = ldexp(1.0 + fr / 1024.0, ex - 15);
    return sign ? -v : v;
}

/* ---- sample access ------------------------------------------------------ */
static double sample_at(const void *plane, int64_t pitch, int bits, int64_t x, int64_t y)
{
    const uint8_t *row = (const uint8_t *)plane + y * pitch;
    if (bits == 8) return (double)row[x];
    uint16_t v;
    memcpy(&v, row + 2 * x, 2);
    return (double)v;
}

static int64_t clampi(int64_t v, int64_t lo, int64_t hi)
{
    return v < lo ? lo : (v > hi ? hi : v);
}

/* ---- reading A5: 4:2:0 -> 4:4:4 bilinear upsample with edge clamp --------
 * CENTER siting: chroma sample i sits at luma coordinate 2i + 1/2 on each
 * axis, so luma sample x sees chroma coordinate u = (x - 1/2)/2.
 * LEFT (MPEG-2) siting: horizontally co-sited with luma column 2i (u = x/2),
 * vertically centred like CENTER (SPEC.md chroma_up_420).
 * Linear interpolation between floor(u) and floor(u)+1 with indices clamped
 * to the plane (edge replication).  The weights (0, 1/4, 1/2, 3/4) are
 * dyadic, so every product and sum below is exact in double. */
enum { OR_CHROMA_CENTER = 0, OR_CHROMA_LEFT = 1 };

static double chroma_up(const void *plane, int64_t pitch, int bits, int siting,
                        int64_t cw, int64_t ch, int64_t x, int64_t y)
{
    double u = (siting == OR_CHROMA_LEFT) ? x / 2.0 : (x - 0.5) / 2.0, v = (y - 0.5) / 2.0;
    int64_t i0 = (int64_t)floor(u), j0 = (int64_t)floor(v);
    double fu = u - (double)i0, fv = v - (double)j0;
    double top = (1.0 - fu) * sample_at(plane, pitch, bits, clampi(i0, 0, cw - 1), clampi(j0, 0, ch - 1))
               + fu * sample_at(plane, pitch, bits, clampi(i0 + 1, 0, cw - 1), clampi(j0, 0, ch - 1));
    double bot = (1.0 - fu) * sample_at(plane, pitch, bits, clampi(i0, 0, cw - 1), clampi(j0 + 1, 0, ch - 1))
               + fu * sample_at(plane, pitch, bits, clampi(i0 + 1, 0, cw - 1), clampi(j0 + 1, 0, ch - 1));
    return (1.0 - fv) * top + fv * bot;
}

/* ---- dequantisation (SPEC.md colorproc.quantize, inverted; readings A2,
 * A11, A15).  Limited: Y' = (c/2^(d-8) - 16)/219, P = (c/2^(d-8) - 128)/224.
 * Full: Y' = c/(2^d - 1), P = (c - 2^(d-1))/(2^d - 1). */
static double deq_luma(double c, int bits, int range)
{
    if (range == OR_LIMITED) return (c / ldexp(1.0, bits - 8) - 16.0) / 219.0;
    return c / (ldexp(1.0, bits) - 1.0);
}

static double deq_chroma(double c, int bits, int range)
{
    if (range == OR_LIMITED) return (c / ldexp(1.0, bits - 8) - 128.0) / 224.0;
    return (c - ldexp(1.0, bits - 1)) / (ldexp(1.0, bits) - 1.0);
}

/* ---- quantisation (north_star: "scale, round-half-even and clamp"; SPEC.md
 * colorproc.quantize with readings A2 (full-range chroma offset), A3 (RNE),
 * A4 (clamp only the final code to [0, 2^d-1])). */
static double quant_finish(double q, int bits)
{
    double maxc = ldexp(1.0, bits) - 1.0;
    if (isnan(q)) return 0.0;
    if (q >= maxc) return maxc;      /* also +inf */
    if (q <= 0.0) return 0.0;        /* also -inf */
    return nearbyint(q);             /* FE_TONEAREST: ties to even */
}

static double quant_luma(double y, int bits, int range)
{
    double q = (range == OR_LIMITED) ? (219.0 * y + 16.0) * ldexp(1.0, bits - 8)
                                     : (ldexp(1.0, bits) - 1.0) * y;
    return quant_finish(q, bits);
}

static double quant_chroma(double p, int bits, int range)
{
    double q = (range == OR_LIMITED) ? (224.0 * p + 128.0) * ldexp(1.0, bits - 8)
                                     : (ldexp(1.0, bits) - 1.0) * p + ldexp(1.0, bits - 1);
    return quant_finish(q, bits);
}

static void store_sample(void *plane, int64_t pitch, int bits, int64_t x, int64_t y, double code)
{
    uint8_t *row = (uint8_t *)plane + y * pitch;
    if (bits == 8) { row[x] = (uint8_t)code; return; }
    uint16_t v = (uint16_t)code;
    memcpy(row + 2 * x, &v, 2);
}

static void store_tensor(void *t, int dtype, int64_t idx, double v)
{
    if (dtype == OR_F32) { float f = (float)v; memcpy((char *)t + 4 * idx, &f, 4); }
    else { uint16_t h = oracle_half_from_double(v); memcpy((char *)t + 2 * idx, &h, 2); }
}

static double load_tensor(const void *t, int dtype, int64_t idx)
{
    if (dtype == OR_F32) { float f; memcpy(&f, (const char *)t + 4 * idx, 4); return (double)f; }
    uint16_t h; memcpy(&h, (const char *)t + 2 * idx, 2);
    return oracle_double_from_half(h);
}

static int check_format(const oracle_format *f)
{
    if (!f || f->width < 1 || f->height < 1) return -1;
    if (f->bits != 8 && f->bits != 10 && f->bits != 16) return -1;
    if (f->family < OR_YUV420 || f->family > OR_RGB) return -1;
    if (f->range != OR_LIMITED && f->range != OR_FULL) return -1;
    if (f->family == OR_YUV420 && ((f->width & 1) || (f->height & 1))) return -1;
    double kr, kb;
    if (f->family != OR_RGB && kr_kb(f->matrix, &kr, &kb)) return -1;
    return 0;
}

/* ---- frames -> tensor (north_star "frames->tensor"; §3.1 RGB/YUV
 * network I/O and colourspace; §3.3 "same input from different batch placed
 * at contiguous location").
 *
 * planes[3*t + p], pitches[3*t + p]: plane p (Y,U,V or R,G,B) of slot t's
 * frame (duplicates allowed).  Output: NCHW [1, 3N, Hp, Wp]; slot t occupies
 * channels 3t, 3t+1, 3t+2 = R', G', B' (reading A7).  Pixels outside W x H
 * (the alignment padding, reading A6) take the values of the clamped
 * position, i.e. they replicate the last row / column. */
int oracle_f2t_sited(const oracle_format *f, int siting, int N, const void *const *planes,
                     const int64_t *pitches, int64_t Hp, int64_t Wp, int dtype, void *out)
{
    if (siting != OR_CHROMA_CENTER && siting != OR_CHROMA_LEFT) return -1;
    if (check_format(f) || N < 1 || Hp < f->height || Wp < f->width) return -1;
    if (dtype != OR_F32 && dtype != OR_F16) return -1;
    double kr = 0, kb = 0;
    if (f->family != OR_RGB) kr_kb(f->matrix, &kr, &kb);
    int64_t W = f->width, H = f->height, cw = W / 2, ch = H / 2;
    int64_t plane_elems = Hp * Wp;
    for (int t = 0; t < N; ++t) {
        const void *p0 = planes[3 * t], *p1 = planes[3 * t + 1], *p2 = planes[3 * t + 2];
        int64_t s0 = pitches[3 * t], s1 = pitches[3 * t + 1], s2 = pitches[3 * t + 2];
        for (int64_t y = 0; y < Hp; ++y) {
            for (int64_t x = 0; x < Wp; ++x) {
                int64_t xc = x < W ? x : W - 1, yc = y < H ? y : H - 1;
                double r, g, b;
                if (f->family == OR_RGB) {
                    /* reading A15: every channel by the luma rule, no matrix */
                    r = deq_luma(sample_at(p0, s0, f->bits, xc, yc), f->bits, f->range);
                    g = deq_luma(sample_at(p1, s1, f->bits, xc, yc), f->bits, f->range);
                    b = deq_luma(sample_at(p2, s2, f->bits, xc, yc), f->bits, f->range);
                } else {
                    double cy = sample_at(p0, s0, f->bits, xc, yc), cu, cv;
                    if (f->family == OR_YUV420) {
                        cu = chroma_up(p1, s1, f->bits, siting, cw, ch, xc, yc);
                        cv = chroma_up(p2, s2, f->bits, siting, cw, ch, xc, yc);
                    } else {
                        cu = sample_at(p1, s1, f->bits, xc, yc);
                        cv = sample_at(p2, s2, f->bits, xc, yc);
                    }
                    double Y = deq_luma(cy, f->bits, f->range);
                    double Pb = deq_chroma(cu, f->bits, f->range);
                    double Pr = deq_chroma(cv, f->bits, f->range);
                    /* inverse of  Y' = Kr R + (1-Kr-Kb) G + Kb B,
                     *             Pb = (B - Y')/(2(1-Kb)), Pr = (R - Y')/(2(1-Kr))
                     * (SPEC.md colorproc rgb_to_yuv444 / yuv444_to_rgb); no
                     * clamp of R', G', B' (reading A4). */
                    r = Y + 2.0 * (1.0 - kr) * Pr;
                    b = Y + 2.0 * (1.0 - kb) * Pb;
                    /* G' = (Y' - Kr R' - Kb B')/(1-Kr-Kb), written in the
                     * algebraically identical difference form so that the
                     * gray axis (Pb = Pr = 0) is exact (reading A16) */
                    g = Y - (kr * (r - Y) + kb * (b - Y)) / (1.0 - kr - kb);
                }
                int64_t base = (int64_t)(3 * t) * plane_elems + y * Wp + x;
                store_tensor(out, dtype, base, r);
                store_tensor(out, dtype, base + plane_elems, g);
                store_tensor(out, dtype, base + 2 * plane_elems, b);
            }
        }
    }
    return 0;
}

/* Pb, Pr of tensor pixel (x, y) of the output slot whose channels start at
 * cbase: Y' = G + Kr (R - G) + Kb (B - G), Pb = (B - Y')/(2(1 - Kb)),
 * Pr = (R - Y')/(2(1 - Kr)). */
static void pixel_pbpr(const void *tensor, int dtype, int64_t cbase, int64_t plane_elems, int64_t tw,
                       int64_t x, int64_t y, double kr, double kb, double *pb, double *pr)
{
    double R = load_tensor(tensor, dtype, cbase + y * tw + x);
    double G = load_tensor(tensor, dtype, cbase + plane_elems + y * tw + x);
    double B = load_tensor(tensor, dtype, cbase + 2 * plane_elems + y * tw + x);
    double Y = G + kr * (R - G) + kb * (B - G);
    *pb = (B - Y) / (2.0 * (1.0 - kb));
    *pr = (R - Y) / (2.0 * (1.0 - kr));
}

/* ---- tensor -> frames (north_star "tensor->frames": "RGB->YUV matrix,
 * chroma downsampling, scale, round-half-even and clamp").
 *
 * tensor: NCHW [1, 3M, th, tw]; output slot o reads channels 3o..3o+2 of the
 * top-left Ho x Wo window (Ho, Wo = the output frame size, §3.2
 * scale factor).  planes[3*o + p], pitches[3*o + p]: output planes.
 *   Y' = G + Kr (R - G) + Kb (B - G)                 (exact on the gray axis)
 *   Pb = (B - Y') / (2 (1 - Kb)),  Pr = (R - Y') / (2 (1 - Kr))   (division)
 *   4:2:0: Pb, Pr of the 2x2 block {(2i,2j),(2i+1,2j),(2i,2j+1),(2i+1,2j+1)}
 *          averaged as ((a + b) + (c + d)) / 4  (reading A5 centre siting, A13)
 *   quantise (limited/full, readings A2/A3/A4). */
int oracle_t2f_sited(const oracle_format *fo, int siting, int M, const void *tensor, int dtype,
                     int64_t th, int64_t tw, void *const *planes, const int64_t *pitches)
{
    if (siting != OR_CHROMA_CENTER && siting != OR_CHROMA_LEFT) return -1;
    if (check_format(fo) || M < 1 || th < fo->height || tw < fo->width) return -1;
    if (dtype != OR_F32 && dtype != OR_F16) return -1;
    double kr = 0, kb = 0;
    if (fo->family != OR_RGB) kr_kb(fo->matrix, &kr, &kb);
    int64_t Wo = fo->width, Ho = fo->height, plane_elems = th * tw;
    int bits = fo->bits, range = fo->range;
    int old_round = fegetround();
    fesetround(FE_TONEAREST);
    for (int o = 0; o < M; ++o) {
        void *p0 = planes[3 * o], *p1 = planes[3 * o + 1], *p2 = planes[3 * o + 2];
        int64_t s0 = pitches[3 * o], s1 = pitches[3 * o + 1], s2 = pitches[3 * o + 2];
        int64_t cbase = (int64_t)(3 * o) * plane_elems;
        for (int64_t y = 0; y < Ho; ++y) {
            for (int64_t x = 0; x < Wo; ++x) {
                double R = load_tensor(tensor, dtype, cbase + y * tw + x);
                double G = load_tensor(tensor, dtype, cbase + plane_elems + y * tw + x);
                double B = load_tensor(tensor, dtype, cbase + 2 * plane_elems + y * tw + x);
                if (fo->family == OR_RGB) {
                    store_sample(p0, s0, bits, x, y, quant_luma(R, bits, range));
                    store_sample(p1, s1, bits, x, y, quant_luma(G, bits, range));
                    store_sample(p2, s2, bits, x, y, quant_luma(B, bits, range));
                    continue;
                }
                double Y = G + kr * (R - G) + kb * (B - G);
                store_sample(p0, s0, bits, x, y, quant_luma(Y, bits, range));
                if (fo->family == OR_YUV444) {
                    double Pb = (B - Y) / (2.0 * (1.0 - kb));
                    double Pr = (R - Y) / (2.0 * (1.0 - kr));
                    store_sample(p1, s1, bits, x, y, quant_chroma(Pb, bits, range));
                    store_sample(p2, s2, bits, x, y, quant_chroma(Pr, bits, range));
                }
            }
        }
        if (fo->family != OR_YUV420) continue;
        for (int64_t j = 0; j < Ho / 2; ++j) {
            for (int64_t i = 0; i < Wo / 2; ++i) {
                double mb, mr;
                if (siting == OR_CHROMA_CENTER) {
                    double pb[4], pr[4];
                    for (int k = 0; k < 4; ++k) {
                        int64_t x = 2 * i + (k & 1), y = 2 * j + (k >> 1);
                        pixel_pbpr(tensor, dtype, cbase, plane_elems, tw, x, y, kr, kb, &pb[k], &pr[k]);
                    }
                    mb = ((pb[0] + pb[1]) + (pb[2] + pb[3])) / 4.0;
                    mr = ((pr[0] + pr[1]) + (pr[2] + pr[3])) / 4.0;
                } else {
                    /* LEFT (MPEG-2): chroma i sits on luma column 2i and
                     * between rows 2j and 2j+1: per row the [1,2,1]/4
                     * low-pass at column 2i (column 2i-1 clamped to 0),
                     * then the mean of the two rows (reading A5). */
                    double hb[2], hr[2];
                    for (int r = 0; r < 2; ++r) {
                        double b3[3], r3[3];
                        for (int k = 0; k < 3; ++k) {
                            int64_t x = clampi(2 * i - 1 + k, 0, Wo - 1);
                            pixel_pbpr(tensor, dtype, cbase, plane_elems, tw, x, 2 * j + r, kr, kb, &b3[k], &r3[k]);
                        }
                        hb[r] = (b3[0] + 2.0 * b3[1]) + b3[2];
                        hr[r] = (r3[0] + 2.0 * r3[1]) + r3[2];
                    }
                    mb = (hb[0] + hb[1]) / 8.0;
                    mr = (hr[0] + hr[1]) / 8.0;
                }
                store_sample(p1, s1, bits, i, j, quant_chroma(mb, bits, range));
                store_sample(p2, s2, bits, i, j, quant_chroma(mr, bits, range));
            }
        }
    }
    fesetround(old_round);
    return 0;
}

int oracle_f2t(const oracle_format *f, int N, const void *const *planes,
               const int64_t *pitches, int64_t Hp, int64_t Wp, int dtype, void *out)
{
    return oracle_f2t_sited(f, OR_CHROMA_CENTER, N, planes, pitches, Hp, Wp, dtype, out);
}

int oracle_t2f(const oracle_format *fo, int M, const void *tensor, int dtype,
               int64_t th, int64_t tw, void *const *planes, const int64_t *pitches)
{
    return oracle_t2f_sited(fo, OR_CHROMA_CENTER, M, tensor, dtype, th, tw, planes, pitches);
}

/* ---- YUV-native network tensors (§3.1: "NNVISR supports
 * input and output in both RGB and YUV pixel format ... YUV420 halves the
 * spatial dimension of 2 in 3 of its channels").
 * No matrix and no resampling: the network sees the clip's own planes,
 * dequantised.  Reading A22: Y' in [0, 1] and U = Pb + 1/2, V = Pr + 1/2 in
 * [0, 1] (SPEC.md VideoFrame float planes, "(Y,U,V) = (1,0.5,0.5) -> white",
 * S:336-337).
 *
 * Tensors: luma [N, Hp, Wp] (slot t = channel t) and chroma [2N, Hc, Wc]
 * (slot t = channels 2t (U), 2t+1 (V)); Hc, Wc = Hp/2, Wp/2 for 4:2:0, else
 * Hp, Wp.  Padding replicates the last row / column of each plane (reading
 * A6 applied per plane).  RGB clips are rejected. */
int oracle_f2t_yuv(const oracle_format *f, int N, const void *const *planes, const int64_t *pitches,
                   int64_t Hp, int64_t Wp, int dtype, void *luma, void *chroma)
{
    if (check_format(f) || f->family == OR_RGB || N < 1 || Hp < f->height || Wp < f->width) return -1;
    if (dtype != OR_F32 && dtype != OR_F16) return -1;
    int sub = f->family == OR_YUV420;
    if (sub && ((Hp | Wp) & 1)) return -1;
    int64_t W = f->width, H = f->height, cw = sub ? W / 2 : W, ch = sub ? H / 2 : H;
    int64_t Hc = sub ? Hp / 2 : Hp, Wc = sub ? Wp / 2 : Wp;
    for (int t = 0; t < N; ++t) {
        for (int64_t y = 0; y < Hp; ++y)
            for (int64_t x = 0; x < Wp; ++x) {
                double c = sample_at(planes[3 * t], pitches[3 * t], f->bits, x < W ? x : W - 1, y < H ? y : H - 1);
                store_tensor(luma, dtype, ((int64_t)t * Hp + y) * Wp + x, deq_luma(c, f->bits, f->range));
            }
        for (int k = 0; k < 2; ++k)
            for (int64_t y = 0; y < Hc; ++y)
                for (int64_t x = 0; x < Wc; ++x) {
                    double c = sample_at(planes[3 * t + 1 + k], pitches[3 * t + 1 + k], f->bits,
                                         x < cw ? x : cw - 1, y < ch ? y : ch - 1);
                    store_tensor(chroma, dtype, ((int64_t)(2 * t + k) * Hc + y) * Wc + x,
                                 deq_chroma(c, f->bits, f->range) + 0.5);
                }
    }
    return 0;
}

/* Inverse: luma [M, th, tw], chroma [2M, thc, twc] (thc, twc = th/2, tw/2
 * for 4:2:0, else th, tw); output slot o reads the top-left window of its
 * planes.  Y code = quantise(Y'), chroma code = quantise(U - 1/2) (readings
 * A2-A4, A22). */
int oracle_t2f_yuv(const oracle_format *fo, int M, const void *luma, const void *chroma, int dtype,
                   int64_t th, int64_t tw, void *const *planes, const int64_t *pitches)
{
    if (check_format(fo) || fo->family == OR_RGB || M < 1 || th < fo->height || tw < fo->width) return -1;
    if (dtype != OR_F32 && dtype != OR_F16) return -1;
    int sub = fo->family == OR_YUV420;
    if (sub && ((th | tw) & 1)) return -1;
    int64_t Wo = fo->width, Ho = fo->height, cw = sub ? Wo / 2 : Wo, ch = sub ? Ho / 2 : Ho;
    int64_t thc = sub ? th / 2 : th, twc = sub ? tw / 2 : tw;
    int old_round = fegetround();
    fesetround(FE_TONEAREST);
    for (int o = 0; o < M; ++o) {
        for (int64_t y = 0; y < Ho; ++y)
            for (int64_t x = 0; x < Wo; ++x) {
                double v = load_tensor(luma, dtype, ((int64_t)o * th + y) * tw + x);
                store_sample(planes[3 * o], pitches[3 * o], fo->bits, x, y, quant_luma(v, fo->bits, fo->range));
            }
        for (int k = 0; k < 2; ++k)
            for (int64_t y = 0; y < ch; ++y)
                for (int64_t x = 0; x < cw; ++x) {
                    double v = load_tensor(chroma, dtype, ((int64_t)(2 * o + k) * thc + y) * twc + x);
                    store_sample(planes[3 * o + 1 + k], pitches[3 * o + 1 + k], fo->bits, x, y,
                                 quant_chroma(v - 0.5, fo->bits, fo->range));
                }
    }
    fesetround(old_round);
    return 0;
}

/* ---- scalar helpers exposed for the closed-form / invariant pins -------- */
int oracle_rgb_to_codes(int matrix, int bits, int range, double R, double G, double B,
                        double *cy, double *cb, double *cr)
{
    double kr, kb;
    if (kr_kb(matrix, &kr, &kb)) return -1;
    int old = fegetround();
    fesetround(FE_TONEAREST);
    double Y = G + kr * (R - G) + kb * (B - G);
    *cy = quant_luma(Y, bits, range);
    *cb = quant_chroma((B - Y) / (2.0 * (1.0 - kb)), bits, range);
    *cr = quant_chroma((R - Y) / (2.0 * (1.0 - kr)), bits, range);
    fesetround(old);
    return 0;
}

int oracle_codes_to_rgb(int matrix, int bits, int range, double cy, double cb, double cr,
                        double *R, double *G, double *B)
{
    double kr, kb;
    if (kr_kb(matrix, &kr, &kb)) return -1;
    double Y = deq_luma(cy, bits, range), Pb = deq_chroma(cb, bits, range),
           Pr = deq_chroma(cr, bits, range);
    *R = Y + 2.0 * (1.0 - kr) * Pr;
    *B = Y + 2.0 * (1.0 - kb) * Pb;
    *G = Y - (kr * (*R - Y) + kb * (*B - Y)) / (1.0 - kr - kb);
    return 0;
}

/* ---- scene-change detection (SPEC.md [MODULE] scenedetect,
 * detect_scene_changes).
 * The paper delegates detection to upstream filters (§3.2
 * P:333-339); this is the SPEC's detector: frame i (i > 0) starts a scene
 * iff the mean absolute luma difference to frame i-1, on the normalised
 * luma scale, exceeds the threshold.  Luma = the Y plane; for RGB clips
 * 0.299 R + 0.587 G + 0.114 B, kept exact as the integer 299R + 587G + 114B
 * (units of 1/1000 code).  Normalisation: one code step is 1/(219*2^(d-8))
 * (limited) or 1/(2^d-1) (full), the dequantisation of reading A2.
 * sad[i] = sum over pixels of |luma_i - luma_{i-1}| (exact integer, in the
 * units above); mad = sad / (pixels * scale [* 1000 for RGB]); cut = mad > t.
 * frames[i] = 3 plane pointers + pitches of frame i; sad[0] = cut[0] = 0. */
int oracle_scene_detect(const oracle_format *f, int count, const void *const *planes, const int64_t *pitches,
                        double threshold, uint64_t *sad, uint8_t *cut)
{
    if (check_format(f) || count < 0) return -1;
    int64_t W = f->width, H = f->height;
    double scale = (f->range == OR_LIMITED) ? 219.0 * ldexp(1.0, f->bits - 8) : ldexp(1.0, f->bits) - 1.0;
    if (f->family == OR_RGB) scale *= 1000.0;
    for (int i = 0; i < count; ++i) {
        uint64_t s = 0;
        if (i > 0) {
            for (int64_t y = 0; y < H; ++y) {
                for (int64_t x = 0; x < W; ++x) {
                    int64_t a, b;
                    if (f->family == OR_RGB) {
                        a = 299 * (int64_t)sample_at(planes[3 * i], pitches[3 * i], f->bits, x, y) +
                            587 * (int64_t)sample_at(planes[3 * i + 1], pitches[3 * i + 1], f->bits, x, y) +
                            114 * (int64_t)sample_at(planes[3 * i + 2], pitches[3 * i + 2], f->bits, x, y);
                        b = 299 * (int64_t)sample_at(planes[3 * i - 3], pitches[3 * i - 3], f->bits, x, y) +
                            587 * (int64_t)sample_at(planes[3 * i - 2], pitches[3 * i - 2], f->bits, x, y) +
                            114 * (int64_t)sample_at(planes[3 * i - 1], pitches[3 * i - 1], f->bits, x, y);
                    } else {
                        a = (int64_t)sample_at(planes[3 * i], pitches[3 * i], f->bits, x, y);
                        b = (int64_t)sample_at(planes[3 * i - 3], pitches[3 * i - 3], f->bits, x, y);
                    }
                    s += (uint64_t)(a > b ? a - b : b - a);
                }
            }
        }
        sad[i] = s;
        double mad = (double)s / ((double)(W * H) * scale);
        cut[i] = (uint8_t)(i > 0 && mad > threshold);
    }
    return 0;
}
