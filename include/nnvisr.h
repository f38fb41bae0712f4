/*
 * nnvisr.h -- C ABI of the B200-native NNVISR frame<->tensor hot path.
 *
 * What it computes (arXiv 2308.03121, /root/reference/PAPER.md):
 *   - frames -> tensor: assemble the tuple of N consecutive planar integer
 *     frames a network consumes ("a tuple of images", §1; "n ... the
 *     number of frames being consumed by the network for each inference run",
 *     §3.1) into one NCHW RGB tensor, converting pixel format and
 *     colourspace (§3.1);
 *   - tensor -> frames: convert the network's RGB output tensor back to
 *     integer planar frames of the clip's format at the scaled size (§3.2
 *     P:313-328);
 *   - the tuple plan: which frames form each tuple, never crossing a scene
 *     change (§3.2, §3.3).
 * Where the paper is silent the readings A1..A22 of DESIGN.md §3 apply
 * (centre chroma siting, replicate padding, round-half-even, ...).
 *
 * Conventions shared by every call:
 *   - Every function returns nnvisr_status; NNVISR_OK (0) is success.  On
 *     failure nothing was enqueued and nnvisr_last_error() (thread-local)
 *     names the violated requirement.
 *   - Ownership: the caller owns every frame, tensor, stream and host array it
 *     passes; the library never frees or retains caller memory beyond the
 *     call (device work enqueued by a call reads caller device memory when it
 *     runs).  The library owns the handle and the small device/pinned scratch
 *     buffers behind it; nnvisr_close() frees them.
 *   - Device work is enqueued on the caller's CUDA stream (`stream` is a
 *     cudaStream_t passed as void*; NULL = legacy default stream) and the call
 *     returns after enqueueing.  Asynchronous faults surface at the caller's
 *     synchronisation, or as NNVISR_ERR_CUDA from a later call.
 *   - CUDA graphs: the device calls (frames->tensor, tensor->frames, their
 *     batch / store / YUV forms) may be captured (cudaStreamBeginCapture, or
 *     torch.cuda.graph) on `stream`.  A captured call records its launches
 *     with tables of its own (kept until nnvisr_release_graph_tables or
 *     nnvisr_close), so every replay
 *     converts the same runs / outputs, reading the frames and tensors at
 *     the addresses of capture time and the frame table bound at that time.
 *     The graph must not be replayed after nnvisr_close, nor after a
 *     nnvisr_bind_frames call that binds more frames than were bound at
 *     capture (the table may move).  The host-buffer calls are not capturable.
 *   - A handle is bound to the CUDA device that is current at its first
 *     device call; it is used by one host thread at a time.  nnvisr_open,
 *     nnvisr_tensor_shapes, nnvisr_plan*, nnvisr_close and nnvisr_last_error
 *     do not touch the GPU (they work on machines without one).
 *   - Frames: planar, plane order (Y, U, V) or (R, G, B); 8-bit samples are
 *     uint8, 10/16-bit samples are uint16 holding the value in the low bits.
 *     4:2:0 chroma planes are (width/2) x (height/2).  `pitch` is the byte
 *     distance between rows.  Every plane must be readable for rows * pitch
 *     bytes from its pointer, i.e. including the pitch padding after the
 *     last row (the TMA paths round copy windows up to 16-byte groups and may
 *     copy a whole plane as rows * pitch bytes; the padding values are never
 *     used).  Frames and tensors are in device memory unless a parameter
 *     says "host".
 *   - Tensors: NCHW, batch 1, fp32 or fp16, rows contiguous.  Input tensor
 *     [1, 3N, Hp, Wp]: tuple slot t -> channels 3t, 3t+1, 3t+2 = R', G', B'
 *     (reading A7), Hp/Wp = height/width rounded up to `align`, padding
 *     replicates the last row/column (reading A6).  Output tensor
 *     [1, 3M, t_h, t_w] with t_h >= H*sy, t_w >= W*sx; output slot o ->
 *     channels 3o..3o+2, the top-left (H*sy) x (W*sx) window is converted.
 *   - Vector fast paths need 16-byte aligned plane/tensor pointers and
 *     pitches that are multiples of 16 bytes; anything else is still
 *     converted correctly by a scalar path.
 */
#ifndef NNVISR_H
#define NNVISR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    NNVISR_OK = 0,
    NNVISR_ERR_INVALID_CONFIG = 1,  /* nnvisr_open: format/network violates an invariant */
    NNVISR_ERR_INVALID_ARG = 2,     /* null/misaligned pointer, bad size, index out of range */
    NNVISR_ERR_UNSUPPORTED = 3,     /* valid request this build does not implement */
    NNVISR_ERR_OUT_OF_MEMORY = 4,   /* scratch allocation failed */
    NNVISR_ERR_CUDA = 5,            /* a CUDA runtime call or kernel launch failed */
    NNVISR_ERR_NCCL = 6,            /* NCCL missing, or an NCCL call / communicator failed */
    NNVISR_ERR_CAPACITY = 7         /* caller's output array too small */
} nnvisr_status;

/* pixel family */
enum { NNVISR_YUV420 = 0, NNVISR_YUV444 = 1, NNVISR_RGB = 2 };
/* colour matrix (reading A1: ITU Kr, Kb; BT.2020 non-constant luminance) */
enum { NNVISR_BT601 = 0, NNVISR_BT709 = 1, NNVISR_BT2020 = 2 };
/* quantisation range (reading A2) */
enum { NNVISR_LIMITED = 0, NNVISR_FULL = 1 };
/* 4:2:0 chroma siting (reading A5): CENTER = chroma between the 2x2 luma
 * block (bilinear 3/4,1/4 up; 2x2 box mean down); LEFT = MPEG-2, horizontally
 * co-sited with even luma columns, vertically centred (up: 1 | 1/2,1/2
 * horizontally; down: [1,2,1]/4 horizontally, 1/2,1/2 vertically; SPEC.md
 * S:339-347).  Both sitings run on the TMA-pipelined kernels where the
 * geometry allows (16-byte aligned planes, pitches and tensor rows). */
enum { NNVISR_CHROMA_CENTER = 0, NNVISR_CHROMA_LEFT = 1 };
/* tensor element type */
enum { NNVISR_F32 = 0, NNVISR_F16 = 1 };
/* network flags, §3.1 */
enum {
    NNVISR_INTERPOLATION = 1u, /* "Interpolation": output at doubled frame rate */
    NNVISR_EXTRA_FRAME = 2u,   /* "Extra frame": the network takes n+1 frames */
    NNVISR_DOUBLE_FRAME = 4u,  /* "Double frame": 2n outputs per run */
    /* YUV network tensors (§3.1, "NNVISR supports input
     * and output in both RGB and YUV pixel format"; SURVEY.md §8(f) NEXT-3;
     * reading A22).  YUV clips only.  No matrix, no chroma resampling: a
     * YUV tensor pair is a luma tensor [1, K, h, w] (channel k = Y' of slot
     * k, in [0, 1]) and a chroma tensor [1, 2K, hc, wc] (channels 2k, 2k+1 =
     * U = Pb + 1/2, V = Pr + 1/2 of slot k), hc, wc = h/2, w/2 for 4:2:0,
     * else h, w.  Padding replicates the last row / column of each plane. */
    NNVISR_YUV_INPUT = 8u,     /* the network consumes YUV tensors */
    NNVISR_YUV_OUTPUT = 16u    /* the network produces YUV tensors */
};

/* The clip being processed (§3.1: RGB/YUV input, the
 * colourspace the network was trained for). */
typedef struct {
    int32_t width, height;  /* luma samples; even for 4:2:0 */
    int32_t family;         /* NNVISR_YUV420 | NNVISR_YUV444 | NNVISR_RGB */
    int32_t bits;           /* 8 | 10 | 16 */
    int32_t matrix;         /* NNVISR_BT601 | _BT709 | _BT2020 (ignored for RGB) */
    int32_t range;          /* NNVISR_LIMITED | NNVISR_FULL */
    int32_t chroma_loc;     /* NNVISR_CHROMA_CENTER */
} nnvisr_clip_format;

/* The network's tuple contract (§3.1, §3.2).
 * Accepted shapes (anything else is NNVISR_ERR_INVALID_CONFIG):
 *   paper grouping: left_context = 0 (or -1), input_count = n + (EXTRA ? 1 : 0),
 *                   output_count in {n, 2n, 2n+1};
 *   sliding window: no INTERPOLATION / EXTRA / DOUBLE flag, n = 1, output_count = 1, any input_count >= 1,
 *                   left_context L in [0, N) (-1 = (N-1)/2, reading A8).
 * DOUBLE_FRAME requires INTERPOLATION; INTERPOLATION without DOUBLE_FRAME
 * requires scale 1 (SPEC.md model-desc invariants). */
typedef struct {
    int32_t input_count;   /* N, 1..16 */
    int32_t output_count;  /* M, 1..16 */
    int32_t n;             /* frames consumed per run, >= 1 */
    int32_t left_context;  /* L; -1 = default */
    uint32_t flags;        /* NNVISR_INTERPOLATION | _EXTRA_FRAME | _DOUBLE_FRAME */
    int32_t sx_num, sx_den, sy_num, sy_den;  /* rational scale factor; W*sx, H*sy integral */
    int32_t align;         /* input tensor H/W multiple: power of two in [1, 256] */
    int32_t dtype;         /* NNVISR_F32 | NNVISR_F16 (both tensors) */
} nnvisr_network;

/* One frame: three plane pointers and their pitches in bytes. */
typedef struct {
    void *plane[3];
    int64_t pitch[3];
} nnvisr_frame;

typedef struct nnvisr_handle nnvisr_handle;

/* Validate the clip format and network contract and create a handle.
 * *out is set only on success.  Does not touch the GPU. */
nnvisr_status nnvisr_open(const nnvisr_clip_format *format, const nnvisr_network *network,
                          nnvisr_handle **out);

/* Free the handle and its scratch buffers.  nnvisr_close(NULL) is OK.  The
 * caller must make sure no enqueued work of this handle is still pending. */
nnvisr_status nnvisr_close(nnvisr_handle *h);

/* Text of the last failure on this thread ("" if none). */
const char *nnvisr_last_error(void);

/* Input tensor shape [1, 3N, Hp, Wp] and minimum output tensor shape
 * [1, 3M, H*sy, W*sx]; also the output frame size (W*sx, H*sy).  For a YUV
 * side (NNVISR_YUV_INPUT / _OUTPUT) the luma tensor: [1, N, Hp, Wp] /
 * [1, M, H*sy, W*sx]. */
nnvisr_status nnvisr_tensor_shapes(const nnvisr_handle *h, int64_t in_nchw[4], int64_t out_nchw[4]);

/* Chroma tensor shapes of the YUV sides: in [1, 2N, Hc, Wc], out
 * [1, 2M, hc, wc] at the minimum output tensor size; all zeros for an RGB
 * side.
 *
 * Packed layout: every call that takes ONE tensor pointer per tuple (or one
 * store) uses, for a YUV side, the luma planes followed directly by the
 * chroma planes: tuple = [K luma planes][2K chroma planes] (K = N or M), and
 * a store slot (nnvisr_frames_to_store / _to_slots / nnvisr_copy_slot) =
 * [Y][U][V] = Hp*Wp + 2*Hc*Wc elements.  The *_yuv_batch calls take the two
 * tensors separately. */
nnvisr_status nnvisr_chroma_shapes(const nnvisr_handle *h, int64_t in_nchw[4], int64_t out_nchw[4]);

/* Tuple plan of a whole clip (steps A1-A2; §3.3).
 * cut: host [num_frames]; cut[k] != 0 means a scene change between frames
 * k-1 and k (cut[0] ignored; reading A9).  Writes run r's input frame indices
 * to run_inputs[r*N .. r*N+N-1] and its half-open fresh interval to
 * run_fresh[2r], run_fresh[2r+1] (host arrays, capacity `cap` runs);
 * *num_runs = number of runs.  NNVISR_ERR_CAPACITY if cap is too small
 * (*num_runs then holds the required count). */
nnvisr_status nnvisr_plan(const nnvisr_handle *h, int64_t num_frames, const uint8_t *cut,
                          int64_t *run_inputs, int64_t *run_fresh, int64_t cap, int64_t *num_runs);

/* Plan of the runs whose fresh frames lie in [fresh_begin, fresh_end) of a
 * clip of num_frames frames, knowing only the cut flags of the window
 * [first, first+count) (a shard plus its halo).  cut: host
 * [count], cut[i] is the flag of frame first+i.  Requires the window to
 * cover [max(0, fresh_begin-L), min(num_frames, fresh_end+N-1-L)).  For the
 * paper's n > 1 grouping the window must be the whole clip (otherwise
 * NNVISR_ERR_UNSUPPORTED; a shard window uses nnvisr_plan_range_anchored).
 * The result equals nnvisr_plan of the whole clip restricted to those runs. */
nnvisr_status nnvisr_plan_range(const nnvisr_handle *h, int64_t num_frames, int64_t first,
                                int64_t count, const uint8_t *cut, int64_t fresh_begin,
                                int64_t fresh_end, int64_t *run_inputs, int64_t *run_fresh,
                                int64_t cap, int64_t *num_runs);

/* Scene-padded store layout for store mode S (§3.3
 * each frame converted once into a frame-major store whose
 * contiguous slot runs are the tuples -- extended to the tuples with
 * duplicated inputs at scene edges, P:352-358 / reading A8): the position
 * sequence Q concatenates, for each scene [s, e) met by the owned fresh
 * frames, L copies of s, s .. e-1 and R = N-1-L copies of e-1 (only the
 * entries the owned tuples read), so that EVERY tuple k in [fresh_begin,
 * fresh_end) -- at a scene edge too -- is the contiguous window Q[w_k ..
 * w_k+N-1] and nothing is materialised.  positions: host int64 [cap]
 * receives Q (absolute frame indices; convert with nnvisr_frames_to_slots,
 * which reads a repeated frame once); *num_positions = |Q| (NNVISR_ERR_CAPACITY
 * if cap is short, *num_positions then holds the size needed, at most
 * (fresh_end - fresh_begin) + scenes * (N-1)); window_start: host int64
 * [fresh_end - fresh_begin], w_k at [k - fresh_begin].  The window [first,
 * first+count) and its flags cut (host [count], as nnvisr_plan_range) must
 * cover [max(0, fresh_begin-L), min(num_frames, fresh_end+R)).  One fresh
 * frame per tuple (n = 1: sliding windows, or the paper's grouping with
 * n = 1); else NNVISR_ERR_UNSUPPORTED. */
nnvisr_status nnvisr_plan_store(const nnvisr_handle *h, int64_t num_frames, int64_t first, int64_t count,
                                const uint8_t *cut, int64_t fresh_begin, int64_t fresh_end, int64_t *positions,
                                int64_t cap, int64_t *num_positions, int64_t *window_start);

/* Halo a shard's window needs for this handle's plan: a run reads frames
 * base-L .. base-L+N-1 (clamped to its scene) with base <= its first fresh
 * frame lo, and under the paper's grouping with n > 1 the last run of a
 * scene recycles up to n-1 frames before lo (base = max(s, e-n), PAPER.md
 * §3.3).  So *left = L + (paper grouping ? n-1 : 0) frames before
 * the shard and *right = N-1-L after it (the L, R of nnvisr_shard_of /
 * nnvisr_halo_exchange).  Host only. */
nnvisr_status nnvisr_halo_extent(const nnvisr_handle *h, int32_t *left, int32_t *right);

/* nnvisr_plan_range for the paper's grouping with n > 1 on a shard window
 * (SURVEY.md §8(e) "Limitation"): a run's phase lo = s + k*n is counted from
 * its scene start s (§3.3), which may lie many shards to
 * the left, so the window's flags alone do not fix the plan.  scene_start is
 * the start of the scene containing frame fresh_begin (the last k <=
 * fresh_begin with cut[k] = 1, k > 0, else 0; from nnvisr_cut_allgather +
 * nnvisr_scene_start_scan across ranks).  The window [first, first+count)
 * with its flags cut (host [count]) must cover [max(scene_start,
 * fresh_begin-left), min(num_frames, fresh_end+right)) for the handle's
 * nnvisr_halo_extent.  Returns the runs whose first fresh frame lies in
 * [fresh_begin, fresh_end) (the whole clip's plan restricted to them, as
 * nnvisr_plan_range).  NNVISR_ERR_INVALID_ARG if scene_start contradicts
 * the window's flags or the window is too small.  For sliding windows and
 * n = 1 scene_start is ignored and this is nnvisr_plan_range. */
nnvisr_status nnvisr_plan_range_anchored(const nnvisr_handle *h, int64_t num_frames, int64_t first, int64_t count,
                                         const uint8_t *cut, int64_t scene_start, int64_t fresh_begin,
                                         int64_t fresh_end, int64_t *run_inputs, int64_t *run_fresh, int64_t cap,
                                         int64_t *num_runs);

/* Bind the device-resident frames that batched calls refer to: frames[i]
 * (host array of descriptors) is frame number base+i.  The descriptors are
 * copied to a handle-owned device table (synchronously); the pixel data is
 * not copied and must stay valid while batched work referring to it runs.
 * Re-binding replaces the table (after the handle's pending batched work). */
nnvisr_status nnvisr_bind_frames(nnvisr_handle *h, int64_t base, const nnvisr_frame *frames,
                                 int64_t count);

/* frames -> tensor for one tuple (steps A3-A7).  in: host array [N] of frame
 * descriptors (the same frame may appear several times); tensor: device
 * [1, 3N, Hp, Wp] of the handle's dtype, 16-byte aligned. */
nnvisr_status nnvisr_frames_to_tensor(nnvisr_handle *h, const nnvisr_frame *in, void *tensor,
                                      void *stream);

/* frames -> tensor for num_runs tuples in one launch.  run_inputs: host
 * [num_runs * N] absolute frame indices (e.g. from nnvisr_plan), each within
 * the bound table; tuple r is written to tensors + r*tensor_stride_bytes
 * (stride >= the tensor size, multiple of 16). */
nnvisr_status nnvisr_frames_to_tensor_batch(nnvisr_handle *h, const int64_t *run_inputs,
                                            int64_t num_runs, void *tensors,
                                            int64_t tensor_stride_bytes, void *stream);

/* Store mode (SURVEY.md §8(d) "S"; §3.3 P:373-379 at batch 1):
 * convert bound frames first .. first+count-1 once each into a frame-major
 * store of slots [3][Hp][Wp]; slot k = frame first+k at store + k*3*Hp*Wp*elem.
 * A run whose inputs are consecutive indices a, a+1, ..., a+N-1 is then the
 * valid [1, 3N, Hp, Wp] tensor starting at slot (a - first). */
nnvisr_status nnvisr_frames_to_store(nnvisr_handle *h, int64_t first, int64_t count, void *store,
                                     void *stream);

/* tensor -> frames for one tuple's network output (steps B1-B4).  tensor:
 * device [1, 3M, t_h, t_w]; out: host array [M] of output frame descriptors
 * (frames of the clip's family/bits/matrix/range at W*sx x H*sy). */
nnvisr_status nnvisr_tensor_to_frames(nnvisr_handle *h, const void *tensor, int64_t t_h,
                                      int64_t t_w, const nnvisr_frame *out, void *stream);

/* tensor -> frames for `count` output tensors in one launch: tensor c at
 * tensors + c*tensor_stride_bytes; its output slot o goes to out[c*M + o]
 * (host array [count*M] of descriptors). */
nnvisr_status nnvisr_tensor_to_frames_batch(nnvisr_handle *h, const void *tensors,
                                            int64_t tensor_stride_bytes, int64_t t_h,
                                            int64_t t_w, const nnvisr_frame *out, int64_t count,
                                            void *stream);

/* YUV input network (NNVISR_YUV_INPUT): frames -> separate luma and chroma
 * tensors.  Run r's luma [N, Hp, Wp] at luma + r*luma_stride_bytes (16-byte
 * aligned, stride a multiple of 16), its chroma [2N, Hc, Wc] at
 * chroma + r*chroma_stride_bytes (element aligned).  Otherwise as
 * nnvisr_frames_to_tensor_batch.  NNVISR_ERR_INVALID_ARG for an RGB-input
 * handle. */
nnvisr_status nnvisr_frames_to_tensor_yuv_batch(nnvisr_handle *h, const int64_t *run_inputs, int64_t num_runs,
                                                void *luma, int64_t luma_stride_bytes, void *chroma,
                                                int64_t chroma_stride_bytes, void *stream);

/* YUV output network (NNVISR_YUV_OUTPUT): tuple c's luma [M, t_h, t_w] at
 * luma + c*luma_stride_bytes, its chroma [2M, t_h/2, t_w/2] (4:2:0; 4:4:4:
 * [2M, t_h, t_w]) at chroma + c*chroma_stride_bytes; t_h, t_w even for 4:2:0.
 * Output slot o -> out[c*M + o] as nnvisr_tensor_to_frames_batch (plane[0]
 * == NULL: not converted).  NNVISR_ERR_INVALID_ARG for an RGB-output handle. */
nnvisr_status nnvisr_tensor_to_frames_yuv_batch(nnvisr_handle *h, const void *luma, int64_t luma_stride_bytes,
                                                const void *chroma, int64_t chroma_stride_bytes, int64_t t_h,
                                                int64_t t_w, const nnvisr_frame *out, int64_t count, void *stream);

/* ---- Host-buffer calls: the frames live in (pinned) host memory.  The
 * library stages them through two device staging slots per direction and
 * two internal copy streams, so the uploads of call i+1 and the downloads of
 * call i-1 overlap the kernels of call i on `stream`. */

/* frames -> tensor from host frames: host_frames[i] (host plane pointers,
 * pinned memory for asynchronous copies) is frame base+i, i < count; every
 * frame index in run_inputs [num_runs*N] must lie in [base, base+count).
 * The frames are copied to the device, then converted as by
 * nnvisr_frames_to_tensor_batch into the device tensors on `stream`.  The
 * host frames must stay valid until that work has run. */
nnvisr_status nnvisr_frames_to_tensor_batch_host(nnvisr_handle *h, const nnvisr_frame *host_frames, int64_t base,
                                                 int64_t count, const int64_t *run_inputs, int64_t num_runs,
                                                 void *tensors, int64_t tensor_stride_bytes, void *stream);

/* tensor -> frames into host frames: as nnvisr_tensor_to_frames_batch, the
 * output of tensor c slot o landing in host_out[c*M + o] (host plane
 * pointers; plane[0] == NULL = not presented, not converted).  The download
 * runs on an internal stream: call nnvisr_host_fence before synchronising
 * `stream` to read the host frames. */
nnvisr_status nnvisr_tensor_to_frames_batch_host(nnvisr_handle *h, const void *tensors, int64_t tensor_stride_bytes,
                                                 int64_t t_h, int64_t t_w, const nnvisr_frame *host_out, int64_t count,
                                                 void *stream);

/* Make `stream` wait until every host download enqueued so far is complete. */
nnvisr_status nnvisr_host_fence(nnvisr_handle *h, void *stream);

/* ---- Output emission (§3.1 P:251-261:
 * "Interpolation ... produce output video in doubled framerate"; without
 * "Double frame", "input frames are also used as output frames as is, and
 * network outputs are all treated as intermediate frames"; SPEC.md
 * grouper.schedule_outputs).  For run r of nnvisr_plan, entries
 * e in [run_first[r], run_first[r+1]) say which outputs are presented:
 * source[e] >= 0: network output slot; source[e] < 0: pass-through of input
 * slot -source[e]-1; present[e]: presentation index (frame index, or 2t and
 * 2t+1 under INTERPOLATION).  Only fresh frames are emitted (the recycled
 * prefix of a scene's last run is dropped; with M = 2n+1 the trailing
 * enhanced lookahead is dropped).  Every presentation index 0 .. F-1 (2F-1)
 * appears once.  Host arrays; capacities cap_entries, cap_runs+1. */
nnvisr_status nnvisr_schedule_outputs(const nnvisr_handle *h, int64_t num_frames, const uint8_t *cut,
                                      int32_t *source, int64_t *present, int64_t *run_first, int64_t cap_entries,
                                      int64_t cap_runs, int64_t *num_entries, int64_t *num_runs);

/* Pass-through frames: copy bound frames src_frames[i] (host array of frame
 * indices) verbatim into out[i] (host array of device frame descriptors of
 * the clip's size and format), i < count, on `stream`.
 * nnvisr_tensor_to_frames[_batch] skip outputs whose descriptor has
 * plane[0] == NULL, so a dropped network output costs no traffic. */
nnvisr_status nnvisr_copy_frames(nnvisr_handle *h, const int64_t *src_frames, const nnvisr_frame *out, int64_t count,
                                 void *stream);

/* ---- Batched shared frame store (§3.3 P:360-382 and Fig. 1;
 * SURVEY.md §8(f) NEXT-2).  A batch of b interpolation runs of n+1 frames
 * needs only b*n + 1 distinct frames; the store keeps each input slot's b
 * lanes contiguous (the batched network input of slot k is the [b, 3, Hp, Wp]
 * tensor starting at offset(k, 0)) and the next batch needs one slot copy. */

/* Offset of input slot k (0..n) of lane j (0..b-1) in region r of the shared
 * layout (SPEC.md framestore.shared_slot_offset): base = r*n*b; slot 0 ->
 * base + j; slot n -> base + 1 + j; slot k in 1..n-1 -> base + 1 + b +
 * (k-1)*b + j.  Frame f0 + j*n + k sits there.  Returns -1 for bad arguments. */
int64_t nnvisr_shared_slot_offset(int32_t n, int32_t b, int32_t region, int32_t k, int32_t j);

/* Batches of b runs (SPEC.md grouper.plan_batches), paper grouping only
 * (NNVISR_ERR_UNSUPPORTED for sliding windows): each scene's runs in order,
 * b per batch, never mixing scenes; a short last batch repeats its last run
 * in the remaining lanes with emit = 0.  A batch is shared (Fig. 1 layout,
 * b*n + 1 slots) when the network takes the extra frame and all b lanes are
 * runs over consecutive frames f, f+1, ..., f+n stepping by n; else plain
 * (b*N slots, slot k of lane j at offset k*b + j).  Per batch i (host arrays,
 * capacity `cap` batches): shared[i]; lanes[i*b + j] = run index (as in
 * nnvisr_plan); emit[i*b + j]; slot_frames[i*b*N + o] = frame at offset o
 * (-1 past the batch's slot count).  NNVISR_ERR_CAPACITY if cap is short. */
nnvisr_status nnvisr_plan_batches(const nnvisr_handle *h, int64_t num_frames, const uint8_t *cut, int32_t b,
                                  uint8_t *shared, int64_t *lanes, uint8_t *emit, int64_t *slot_frames,
                                  int64_t cap, int64_t *num_batches);

/* frames -> slots of a frame-major store: slot i (3*Hp*Wp elements at
 * store + i*3*Hp*Wp*elem) receives bound frame slot_frames[i] (host array
 * [count]; -1 leaves the slot untouched).  A frame listed at several slots
 * is read and converted once. */
nnvisr_status nnvisr_frames_to_slots(nnvisr_handle *h, const int64_t *slot_frames, int64_t count, void *store,
                                     void *stream);

/* The single-frame advance ("6 to 5 in the figure"):
 * copy store slot src to slot dst on `stream`. */
nnvisr_status nnvisr_copy_slot(nnvisr_handle *h, void *store, int64_t src, int64_t dst, void *stream);

/* Region advance of a bounded store ring (store mode S with a ring of
 * regions; the b = 1 form of PAPER.md P:380-382 "only the
 * last frame need to be copied ... (6 to 5 in the figure)"): copy `count`
 * consecutive slots starting at slot src to slot dst of `store` in one
 * device copy on `stream` (a sliding window of N frames carries its last
 * N-1 slots into the next region).  The two ranges must not overlap
 * (NNVISR_ERR_INVALID_ARG). */
nnvisr_status nnvisr_copy_slots(nnvisr_handle *h, void *store, int64_t src, int64_t dst, int64_t count,
                                void *stream);

/* Scene-change detection (SPEC.md [MODULE] scenedetect,
 * detect_scene_changes, S:105-113 -- the paper leaves detection to upstream
 * filters, §3.2).  For bound frames first+i, i in
 * [0, count): sad[i] = sum over the W x H pixels of |luma(first+i) -
 * luma(first+i-1)|, an exact integer (luma = the Y plane; for RGB clips
 * 299 R + 587 G + 114 B), and cut[i] = 1 iff
 * sad[i] / (W * H * scale) > threshold with scale = 219 * 2^(d-8) (limited)
 * or 2^d - 1 (full), times 1000 for RGB (the normalised luma step of reading
 * A2).  sad[0] = cut[0] = 0: frame first-1 is not compared.  sad (uint64)
 * and cut (uint8) are device arrays [count] written on `stream`; the flags
 * are in the form nnvisr_plan consumes (copy them to the host). */
nnvisr_status nnvisr_scene_detect(nnvisr_handle *h, int64_t first, int64_t count, double threshold,
                                  uint64_t *sad, uint8_t *cut, void *stream);

/* ---- Multi-GPU halo by peer mapping (rank r's tuples
 * near its shard edges read up to L frames owned by rank r-1 and N-1-L
 * frames owned by rank r+1, §3.2 P:347-358 sliding windows).  One
 * process per GPU.  Instead of copying those frames, each rank exports the
 * device buffer that holds its own frames, its neighbours import it, and the
 * halo frames are bound (nnvisr_bind_frames) as descriptors pointing into
 * the neighbour's buffer: the f2t kernels then read them in place, over
 * NVLink between GPUs.  The caller exchanges the handles (e.g. with
 * torch.distributed all_gather_object) and orders the neighbour's writes
 * before the reads (a barrier or an interprocess event), as it would order a
 * copy.  The cut flags of the halo frames are host data and travel with the
 * caller's own exchange. */
typedef struct {
    uint8_t ipc[64];  /* CUDA IPC memory handle of the allocation holding the pointer */
    int64_t offset;   /* the pointer's byte offset inside that allocation */
} nnvisr_peer_handle;

/* Export device pointer dev_ptr (inside any cudaMalloc allocation, e.g. a
 * torch tensor's data_ptr()) of the current process.  The allocation must
 * outlive every importer's use.  NNVISR_ERR_INVALID_ARG for a null or host
 * pointer, NNVISR_ERR_CUDA if the allocation cannot be exported. */
nnvisr_status nnvisr_peer_export(const void *dev_ptr, nnvisr_peer_handle *out);

/* Map an exported buffer of ANOTHER process into this one (on the current
 * device; peer access is enabled lazily) and return the device pointer that
 * corresponds to the exporter's dev_ptr.  Importing a handle in the process
 * that exported it fails with NNVISR_ERR_CUDA (CUDA IPC forbids it). */
nnvisr_status nnvisr_peer_import(const nnvisr_peer_handle *in, void **dev_ptr);

/* Unmap a pointer returned by nnvisr_peer_import (after the work reading it
 * has completed).  NNVISR_ERR_INVALID_ARG for a pointer not imported here. */
nnvisr_status nnvisr_peer_close(void *dev_ptr);

/* ---- Multi-GPU frame-range shards and the NCCL halo exchange (SURVEY.md
 * §8(b), §8(e)).  The clip shards by contiguous frame ranges: rank r of W
 * owns the runs whose fresh frame lies in [r*F/W, (r+1)*F/W).  A sliding
 * window reads L frames before and R = N-1-L frames after its fresh frame
 * (reading A8), and whether each of them is used or replaced by a duplicate
 * depends on its scene-cut flag (§3.2, §3.3).
 * So a rank keeps a WINDOW of frames [left halo | owned | right halo] and
 * needs its neighbours' edge frames and flags: one grouped point-to-point
 * exchange per step, the only data that crosses ranks.  Window rows are
 * frame records of frame_bytes bytes each (a k-frame halo is one message),
 * with the flags in a parallel byte array (cut_window[i] = flag of window
 * frame i, as nnvisr_plan reads it).  The local plan is then
 * nnvisr_plan_range(total, window_first, cut_window, begin, end), which
 * equals the whole clip's plan restricted to the shard.
 *
 * NCCL (libnccl.so.2) is loaded at the first nnvisr_comm_* call (the copy
 * the process already loaded is reused, NNVISR_NCCL_LIB overrides); without
 * it those calls return NNVISR_ERR_NCCL.  nnvisr_shard_of and
 * nnvisr_halo_plan are pure host functions. */

typedef struct {
    int64_t begin, end;               /* owned frames [begin, end) = [r*F/W, (r+1)*F/W) */
    int64_t left, right;              /* halo frames before begin (min(L, begin)) / after end (min(R, F-end)) */
    int64_t window_first, window_count; /* the window = frames [window_first, window_first+window_count) */
} nnvisr_shard;

/* Geometry of shard `rank` of `world` over a clip of `total` frames for a
 * window reaching L frames back and R frames ahead (0 <= L, R <= 15).
 * NNVISR_ERR_INVALID_ARG if rank is outside [0, world) or (world > 1) a
 * shard holds fewer than max(L, R, 1) frames (a halo would then span more
 * than one neighbour). */
nnvisr_status nnvisr_shard_of(int64_t total, int32_t world, int32_t rank, int32_t L, int32_t R, nnvisr_shard *out);

/* One point-to-point message of a rank's halo exchange: window rows
 * [first, first+count) are sent to (send = 1) or received from (send = 0)
 * rank `peer`.  The flags of the same rows travel in a second message of
 * count bytes. */
typedef struct {
    int32_t peer, send;
    int64_t first, count;
} nnvisr_halo_msg;

/* The messages of rank `rank` (at most 4, *count set): my first min(R, F-begin)
 * owned rows to rank-1 and my left halo from it; my last min(L, end) owned
 * rows to rank+1 and my right halo from it.  Every send matches the
 * neighbour's receive of the same count. */
nnvisr_status nnvisr_halo_plan(int64_t total, int32_t world, int32_t rank, int32_t L, int32_t R,
                               nnvisr_halo_msg msgs[4], int32_t *count);

typedef struct nnvisr_comm nnvisr_comm;
#define NNVISR_COMM_ID_BYTES 128

/* A new communicator id (ncclGetUniqueId) on rank 0; broadcast its bytes to
 * the other ranks out of band (e.g. torch.distributed). */
nnvisr_status nnvisr_comm_unique_id(uint8_t id[NNVISR_COMM_ID_BYTES]);

/* One process per GPU: join communicator `id` as rank `rank` of `world` on
 * the CUDA device current in this thread (ncclCommInitRank; collective, every
 * rank must call it).  Free with nnvisr_comm_destroy. */
nnvisr_status nnvisr_comm_init_rank(const uint8_t id[NNVISR_COMM_ID_BYTES], int32_t world, int32_t rank,
                                    nnvisr_comm **out);

/* One process driving ndev GPUs: comms[i] is rank i on device devs[i]
 * (ncclCommInitAll).  Use with nnvisr_halo_exchange_all. */
nnvisr_status nnvisr_comm_init_all(int32_t ndev, const int32_t *devs, nnvisr_comm **comms);

/* Rank, world size and CUDA device of a communicator (any may be NULL). */
nnvisr_status nnvisr_comm_info(const nnvisr_comm *comm, int32_t *rank, int32_t *world, int32_t *device);

/* NNVISR_ERR_NCCL if the communicator has an asynchronous error
 * (ncclCommGetAsyncError: a failed peer or transport); the exchange calls
 * also check after enqueueing. */
nnvisr_status nnvisr_comm_check(const nnvisr_comm *comm);

/* The halo exchange of this rank: one ncclGroupStart /
 * ncclGroupEnd holding the messages of nnvisr_halo_plan(total_frames,
 * world, rank, L, R), each as one ncclSend / ncclRecv of count*frame_bytes
 * bytes of `window` (device, [window_count][frame_bytes], owned rows filled)
 * plus one of count bytes of `cut_window` (device [window_count]), enqueued
 * on `stream`.  window = NULL exchanges the flags only (frames read in place,
 * nnvisr_peer_*); cut_window = NULL the frames only.  Every rank must call it
 * with the same total_frames, L, R.  Returns after enqueueing; the halo rows
 * are valid once `stream` reaches that point.  World 1: nothing to send. */
nnvisr_status nnvisr_halo_exchange(nnvisr_comm *comm, int64_t total_frames, int32_t L, int32_t R, void *window,
                                   int64_t frame_bytes, uint8_t *cut_window, void *stream);

/* Single-process form: the exchange of every rank of an
 * nnvisr_comm_init_all communicator in one group (windows[i],
 * cut_windows[i], streams[i] on device i). */
nnvisr_status nnvisr_halo_exchange_all(nnvisr_comm *const *comms, int32_t ndev, int64_t total_frames, int32_t L,
                                       int32_t R, void *const *windows, int64_t frame_bytes,
                                       uint8_t *const *cut_windows, void *const *streams);

/* The scene-start scan of the paper's n > 1 grouping across ranks
 * (SURVEY.md §8(e) "Limitation": an exclusive scan of the last cut
 * position).  last_cuts: device int64 [world]; on entry element `rank`
 * holds this rank's last cut in its owned frames (nnvisr_last_cut, -1 if
 * none); one in-place ncclAllGather on `stream` fills every element (valid
 * once `stream` reaches that point). */
nnvisr_status nnvisr_cut_allgather(nnvisr_comm *comm, int64_t *last_cuts, void *stream);

/* Host helpers of the scan.  nnvisr_last_cut: the last frame first+i with
 * cut[i] = 1 and first+i > 0 of a host flag array cut [count] (-1 if none;
 * cut[0] of the clip is ignored, reading A9).  nnvisr_scene_start_scan: the
 * start of the scene containing frame `begin` (= this rank's first owned
 * frame) from the gathered last cuts of ranks 0 .. rank-1 (host [world]) and
 * begin's own flag cut_begin: begin if it starts a scene, else the largest
 * lower-rank cut, else 0.  NNVISR_ERR_INVALID_ARG if a lower rank's cut lies
 * at or after begin. */
nnvisr_status nnvisr_last_cut(const uint8_t *cut, int64_t first, int64_t count, int64_t *last_cut);
nnvisr_status nnvisr_scene_start_scan(int32_t world, int32_t rank, const int64_t *last_cuts, int64_t begin,
                                      uint8_t cut_begin, int64_t *scene_start);

/* Free a communicator (ncclCommDestroy; after its work completed).  NULL is OK. */
nnvisr_status nnvisr_comm_destroy(nnvisr_comm *comm);

/* NCCL version code of the loaded library (e.g. 22809), -1 if NCCL is unavailable. */
int32_t nnvisr_nccl_version(void);

/* Free the upload tables of every call captured into a CUDA graph so far
 * (see "CUDA graphs" above).  The caller must have destroyed those graphs
 * (or will never replay them again) and no replay may be in flight; a server
 * that re-captures when its plan changes calls this between captures.  The
 * handle's own ring of upload slots is untouched. */
nnvisr_status nnvisr_release_graph_tables(nnvisr_handle *h);

/* Number of CUDA kernels this library has launched in this process. */
int64_t nnvisr_launch_count(void);

/* Library version string. */
const char *nnvisr_version(void);

#ifdef __cplusplus
}
#endif

#endif /* NNVISR_H */
