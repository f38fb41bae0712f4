// internal.h -- types shared by the C ABI layer (nnvisr.cpp) and the sm_100a
// kernels (kernels.cu).  Not part of the public ABI (include/nnvisr.h).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "nnvisr.h"

struct nnvisr_comm;

namespace nnvisr {

// Set the thread's last-error text (nnvisr_last_error) and return s; defined
// in nnvisr.cpp, used by the other host translation units (comm.cpp).
nnvisr_status set_error(nnvisr_status s, const char *msg);

constexpr int kYUV420 = 0, kYUV444 = 1, kRGB = 2;
constexpr int kF32 = 0, kF16 = 1;
constexpr int kPx = 8;           // luma columns per thread (one 16-byte fp16 store)
constexpr int kThreads = 256;    // CTA size of the conversion kernels

// Device copy of one frame descriptor (same layout as nnvisr_frame).
struct DevFrame {
    const void *plane[3];
    int64_t pitch[3];
};

// frames -> tensor colour constants (steps A5-A6), fp32.
//   luma / RGB channel : v = (16*code - y_off) * y_scale
//   chroma             : P = (s - c_off) * c_scale, s = 16 x the (upsampled) code
//   R = Y + r_pr*Pr ;  B = Y + b_pb*Pb ;  G = Y - g_pb*Pb - g_pr*Pr
//   fp16 tensors: values with |v| < 2^-11 (below which an fp16 ULP is not
//   safely coarser than the fp32 rounding error) are recomputed in fp64 with the *_d constants.
struct F2TColour {
    int32_t y_off, c_off;
    int32_t u_off;  // YUV-native chroma U = P + 1/2 = (16*code - u_off) * c_scale (reading A22)
    float y_scale, c_scale;
    float r_pr, b_pb, g_pb, g_pr;
    float r_v, b_u, g_u, g_v;  // r_pr * c_scale, b_pb * c_scale, g_pb * c_scale, g_pr * c_scale (rounded once)
    double y_scale_d, c_scale_d, r_pr_d, b_pb_d, g_pb_d, g_pr_d;
};

// tensor -> frames colour constants (steps B2-B4), in fp32 and fp64.
//   Y' = G + kr(R-G) + kb(B-G)                      (exact on the gray axis)
//   luma code   = rne(clamp(Y' * ys + yo, 0, maxc))
//   chroma: S = sum over the k pixels of the chroma sample (k = 4 for 4:2:0,
//   1 for 4:4:4) of (B - Y') [or (R - Y')];  P = S / (k * db) by a reciprocal
//   and one FMA correction (correctly rounded, so the primaries' exact 0.5
//   ties stay exact);  chroma code = rne(clamp(P * cs + co, 0, maxc)).
struct T2FColour {
    double kr, kb, db, dr, idb, idr, ys, yo, cs, co, maxc;
    float fkr, fkb, fdb, fdr, fidb, fidr, fys_n, fyo_n, fcs_n, fco_n, fmaxc;  // *_n = / maxc
    // YUV-native chroma (reading A22): code = rne(clamp(U * cs + co2)) with
    // co2 = co - cs/2, i.e. P = U - 1/2 folded into the offset (exact)
    double co2;
};

// frames -> tensor work list of one launch: job j converts the distinct frame
// frames[job_frame[j]] once and stores it to every (run, slot) that uses it:
// dst_code[job_dst[j] .. job_dst[j+1]) = run * 32 + slot, written at
// dst + run * run_stride + slot * slot_bytes.
struct F2TArgs {
    const DevFrame *frames;   // bound frame table (device)
    const int32_t *job_frame; // [jobs] index into `frames`
    const int32_t *job_dst;   // [jobs + 1] CSR offsets into dst_code
    const int32_t *dst_code;  // run * 32 + slot
    char *dst;                // tensor of run 0 of this launch
    int64_t run_stride;       // bytes between consecutive runs' tensors
    int64_t slot_bytes;       // bytes of one slot (3*Hp*Wp*elem)
    int64_t items;            // jobs * units
    int32_t W, H, Hp, Wp;     // clip size and padded tensor size
    int32_t units, col_units; // items per job and column groups per row unit
    int32_t vec_in;           // 1: all bound planes/pitches 16-byte aligned
    int32_t vec_out;          // 1: tensor rows allow 16-byte stores
    // TMA-pipelined path (kernels_tma.cu): tiles = jobs * rowunits * nseg
    int32_t tma_ok, rowunits, nseg, stages, stage_bytes;
    int32_t nob, ob_elems;        // output buffers, elements per buffer
    int32_t band, ls, cs, whole;  // band height (row units), staged row strides, whole-row copies
    int32_t fsegw;                // TMA path: columns per tile segment (kSegW, or the whole row up to 2 x kSegW)
    int32_t nstorers;             // storer threads (1 or 2)
    int32_t cthreads;             // TMA path: converting threads per CTA (multiple of 32, <= kThreads)
    int32_t release_first;        // storers free the next output buffer before (1) or after (0) issuing a tile
    uint64_t *trace;              // experiment timeline buffer (debug & 8)
    int32_t debug;                // experiment switches (NNVISR_F2T_DEBUG), 0 in production
    int64_t pitch_y, pitch_c;     // uniform plane pitches of the bound frames (0 = not uniform)
    int64_t tiles;
    unsigned long long *tile_counter;  // TMA path: zeroed per launch, dynamic tile scheduler
    int64_t jobs, dests;               // distinct frames and (run, slot) destinations of the launch
    F2TColour col;
    // 4:2:0 chroma siting of this launch: 0 centre, 1 LEFT
    int32_t left;
    // YUV-native tensors (NEXT-3, kernels_yuv.cu): the luma of (run, slot) at
    // dst + run*run_stride + slot*slot_bytes ([Hp][Wp]); its chroma planes U,
    // V at dst2 + run*run_stride2 + slot*slot_bytes2 (+ cplane_bytes for V),
    // each [Hc][Wc]
    int32_t yuv, Hc, Wc, vec_out_c;
    char *dst2;
    int64_t run_stride2, slot_bytes2, cplane_bytes;
};

struct T2FArgs {
    const int32_t *job_code;  // optional [jobs]: tuple * 32 + slot (skipped outputs removed); null = dense
    const char *src;          // tensor of job 0's tuple
    int64_t tensor_stride;    // bytes between tuples' tensors
    const DevFrame *out;      // output frame descriptors [count*M] (device)
    int32_t M;                // output slots per tensor
    int64_t items;            // jobs * units
    int32_t Wo, Ho;           // output frame size
    int64_t th, tw;           // tensor spatial size
    int32_t units, col_units;
    int32_t vec_in;           // tensor rows allow 16-byte loads
    int32_t vec_out;          // output planes allow vector stores
    int32_t tma_ok, rowunits, nseg, stages, stage_bytes, segw;
    int32_t cthreads;  // TMA path: consumer threads per CTA (segw / 8 rounded up to warps)
    int32_t lpad;      // TMA path: values staged left of each row segment (LEFT siting), else 0
    int64_t tiles;
    unsigned long long *tile_counter;  // TMA path: zeroed per launch, dynamic tile scheduler
    T2FColour col;
    int32_t left;  // 4:2:0 chroma siting: 0 centre, 1 LEFT
    // YUV-native tensors (NEXT-3): output slot o of tuple c reads luma plane o
    // of src + c*tensor_stride ([th][tw]) and chroma planes 2o, 2o+1 of
    // src2 + c*tensor_stride2 ([thc][twc])
    int32_t yuv, vec_in_c;
    const char *src2;
    int64_t tensor_stride2, thc, twc;
};

// Launchers (kernels.cu).  Return the CUDA error of the launch.
cudaError_t launch_f2t(int family, int bits, int dtype, const F2TArgs &a, cudaStream_t s);
cudaError_t launch_t2f(int family, int bits, int dtype, const T2FArgs &a, cudaStream_t s);
cudaError_t launch_f2t_tma(int family, int bits, int dtype, const F2TArgs &a, cudaStream_t s);
cudaError_t launch_f2t_strip(int bits, int dtype, const F2TArgs &a, cudaStream_t s);
bool f2t_strip_ok(int dtype, const F2TArgs &a);
cudaError_t launch_t2f_tma(int family, int bits, int dtype, const T2FArgs &a, cudaStream_t s);
cudaError_t launch_f2t_yuv(int family, int bits, int dtype, const F2TArgs &a, cudaStream_t s);
cudaError_t launch_f2t_yuv_tma(int family, int bits, int dtype, const F2TArgs &a, cudaStream_t s);
cudaError_t launch_t2f_yuv_tma(int family, int bits, int dtype, const T2FArgs &a, cudaStream_t s);
cudaError_t launch_t2f_yuv(int family, int bits, int dtype, const T2FArgs &a, cudaStream_t s);

cudaError_t launch_scene_detect(int family, int bits, int range, int W, int H, const DevFrame *frames, int count,
                                int vec, double threshold, uint64_t *sad, uint8_t *cut, cudaStream_t s);

void count_launch();

}  // namespace nnvisr
