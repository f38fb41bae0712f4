// hbm_probe.cu -- HBM bandwidth of simple streaming kernels with different
// read:write mixes on this GPU (128-bit loads/stores, grid = 4 x 148 x 256).
// Context for the f2t (write-heavy, ~1:6) and t2f (read-heavy, ~2:1) rooflines.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/hbm_probe.cu -o /tmp/hbm_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void mix(const uint4 *__restrict__ in, uint4 *__restrict__ out, long n_in, int wmul, long n_out)
{
    // each thread reads in[i] (if i < n_in) and writes it to wmul destinations
    const long stride = (long)gridDim.x * blockDim.x;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n_out / wmul; i += stride) {
        uint4 v = i < n_in ? in[i] : make_uint4(i, i, i, i);
        for (int k = 0; k < wmul; ++k) out[(long)k * (n_out / wmul) + i] = v;
    }
}

__global__ void r2w1(const uint4 *__restrict__ in, uint4 *__restrict__ out, long m)
{
    const long stride = (long)gridDim.x * blockDim.x;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
        uint4 x = in[i], y = in[i + m];
        out[i] = make_uint4(x.x ^ y.x, x.y ^ y.y, x.z ^ y.z, x.w ^ y.w);
    }
}

// 1 read : W writes, each CTA-iteration loads a 64 KB chunk into registers
// and writes it to the W destinations one after another (64 KB contiguous each)
template <int W>
__global__ void fanout_chunked(const uint4 *__restrict__ in, uint4 *__restrict__ out, long m)
{
    constexpr int U = 16;
    const long chunk = (long)blockDim.x * U;
    for (long base = (long)blockIdx.x * chunk; base < m; base += (long)gridDim.x * chunk) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long i = base + u * blockDim.x + threadIdx.x;
            v[u] = i < m ? in[i] : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < W; ++k)
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long i = base + u * blockDim.x + threadIdx.x;
                if (i < m) out[(long)k * m + i] = v[u];
            }
    }
}

// same, but the CTA stages the chunk in shared memory and one thread writes it
// to the W destinations with TMA bulk stores (cp.async.bulk.global.shared::cta)
template <int W, int U = 16>
__global__ void fanout_tma(const uint4 *__restrict__ in, uint4 *__restrict__ out, long m)
{
    extern __shared__ __align__(128) uint4 sm[];
    const long chunk = (long)blockDim.x * U;
    for (long base = (long)blockIdx.x * chunk; base < m; base += (long)gridDim.x * chunk) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long i = base + u * blockDim.x + threadIdx.x;
            sm[u * blockDim.x + threadIdx.x] = i < m ? in[i] : make_uint4(0, 0, 0, 0);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            const long n = min(chunk, m - base);
            for (int k = 0; k < W; ++k) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + (long)k * m + base),
                             "r"((unsigned)__cvta_generic_to_shared(sm)), "r"((unsigned)(n * 16))
                             : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// 1 read : W writes with U independent 16-byte loads in flight per thread
// (chunks of U x blockDim vectors; each written to W destinations)
template <int W, int U>
__global__ void fanout_ilp(const uint4 *__restrict__ in, uint4 *__restrict__ out, long m)
{
    const long chunk = (long)blockDim.x * U;
    for (long base = (long)blockIdx.x * chunk; base < m; base += (long)gridDim.x * chunk) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long i = base + u * blockDim.x + threadIdx.x;
            v[u] = i < m ? __ldcs(in + i) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < W; ++k)
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long i = base + u * blockDim.x + threadIdx.x;
                if (i < m) out[(long)k * m + i] = v[u];
            }
    }
}

// 1 read : W writes at strip-kernel occupancy: every warp moves 512-byte
// rows; STG (BULK = false) or per-warp bulk stores of 512 B from a
// double-buffered staging area (BULK = true)
template <int W, bool BULK>
__global__ void __launch_bounds__(256, 2) warp_rows(const uint4 *__restrict__ in, uint4 *__restrict__ out, long m)
{
    __shared__ __align__(128) uint4 stage[8][2][W][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long warps = (long)gridDim.x * 8;
    int b = 0;
    for (long r = (long)blockIdx.x * 8 + w; r * 32 < m; r += warps) {
        const long i = r * 32 + lane;
        const uint4 v = __ldcs(in + i);
        if (!BULK) {
#pragma unroll
            for (int k = 0; k < W; ++k) out[(long)k * m + i] = v;
        } else {
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
#pragma unroll
            for (int k = 0; k < W; ++k) stage[w][b][k][lane] = v;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
#pragma unroll
                for (int k = 0; k < W; ++k)
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;" ::"l"(out + (long)k * m + r * 32),
                                 "r"((unsigned)__cvta_generic_to_shared(&stage[w][b][k][0]))
                                 : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            b ^= 1;
        }
    }
    if (BULK && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void readonly(const uint4 *__restrict__ in, long n, unsigned *sink)
{
    const long stride = (long)gridDim.x * blockDim.x;
    unsigned acc = 0;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        uint4 v = in[i];
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

// 2 reads : 1 write as t2f moves it: inputs staged by TMA bulk copies into a
// ring of S stages (completion on mbarriers, one elected thread issues), the
// result written either by every thread with STG.128 (BULK = false, t2f's
// code stores) or staged in shared memory and written by one thread with TMA
// bulk stores (BULK = true).  Chunk = 256 threads x U vectors per input.
__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
template <bool BULK, int U = 2, int S = 3>
__global__ void __launch_bounds__(256) r2w1_tma(const uint4 *__restrict__ in, uint4 *__restrict__ out, long m)
{
    extern __shared__ __align__(128) uint4 sm[];
    __shared__ __align__(8) unsigned long long full[S];
    constexpr int C = 256 * U;  // vectors per input chunk
    uint4 *stage = sm;          // [S][2][C]
    uint4 *ob = sm + S * 2 * C; // [2][C] (BULK)
    const long nchunks = m / C;
    if (threadIdx.x == 0) {
        for (int k = 0; k < S; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[k])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](long c, int k) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[k])), "r"(2 * C * 16) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(stage + (k * 2) * C)),
                     "l"(in + c * C), "r"(C * 16), "r"(su32(&full[k])) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(stage + (k * 2 + 1) * C)),
                     "l"(in + m + c * C), "r"(C * 16), "r"(su32(&full[k])) : "memory");
    };
    long c0 = blockIdx.x;
    const long G = gridDim.x;
    if (threadIdx.x == 0)
        for (int k = 0; k < S; ++k)
            if (c0 + k * G < nchunks) issue(c0 + k * G, k);
    int k = 0;
    unsigned ph = 0;
    int ob_i = 0;
    for (long c = c0; c < nchunks; c += G) {
        asm volatile("{ .reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W; }" ::"r"(su32(&full[k])), "r"(ph) : "memory");
        const uint4 *x = stage + (k * 2) * C, *y = stage + (k * 2 + 1) * C;
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint4 a = x[u * 256 + threadIdx.x], b = y[u * 256 + threadIdx.x];
            r[u] = make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w);
        }
        __syncthreads();  // every thread has read stage k
        if (threadIdx.x == 0 && c + S * G < nchunks) issue(c + S * G, k);
        if (!BULK) {
#pragma unroll
            for (int u = 0; u < U; ++u) out[c * C + u * 256 + threadIdx.x] = r[u];
        } else {
            if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncthreads();
            uint4 *o = ob + ob_i * C;
#pragma unroll
            for (int u = 0; u < U; ++u) o[u * 256 + threadIdx.x] = r[u];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (threadIdx.x == 0) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + c * C), "r"(su32(o)), "r"(C * 16) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            ob_i ^= 1;
        }
        if (++k == S) { k = 0; ph ^= 1; }
    }
    if (BULK && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char **argv)
{
    const long bytes = 4l << 30;
    const long n = bytes / 16;
    uint4 *a, *b;
    unsigned *sink;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(a, 1, bytes);
    cudaEvent_t s, e;
    cudaEventCreate(&s);
    cudaEventCreate(&e);
    const int grid = 4 * 148, block = 256;
    auto run = [&](const char *name, auto fn, double moved) {
        for (int i = 0; i < 3; ++i) fn();
        float best = 1e9;
        for (int r = 0; r < 10; ++r) {
            cudaEventRecord(s);
            fn();
            cudaEventRecord(e);
            cudaEventSynchronize(e);
            float ms;
            cudaEventElapsedTime(&ms, s, e);
            if (ms < best) best = ms;
        }
        printf("{\"probe\": \"%s\", \"gbs\": %.1f}\n", name, moved / (best / 1000) / 1e9);
    };
    if (argc > 1) {  // t2f-shaped 2R:1W probes only: hbm_probe t2f
        auto tma = [&](auto kern, const char *name, int U, int S, int per_sm, bool bulk) {
            const int smem = (S * 2 + (bulk ? 2 : 0)) * 256 * U * 16;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            run(name, [&] { kern<<<per_sm * 148, 256, smem>>>(a, b, n / 2); }, 1.5 * bytes);
        };
        run("2r_1w", [&] { r2w1<<<grid, block>>>(a, b, n / 2); }, 1.5 * bytes);
        tma(r2w1_tma<false, 2, 3>, "2r_1w_tma_stg_U2_S3_x3", 2, 3, 3, false);
        tma(r2w1_tma<true, 2, 3>, "2r_1w_tma_bulk_U2_S3_x3", 2, 3, 3, true);
        tma(r2w1_tma<false, 4, 3>, "2r_1w_tma_stg_U4_S3_x2", 4, 3, 2, false);
        tma(r2w1_tma<true, 4, 3>, "2r_1w_tma_bulk_U4_S3_x2", 4, 3, 2, true);
        tma(r2w1_tma<false, 2, 4>, "2r_1w_tma_stg_U2_S4_x3", 2, 4, 3, false);
        tma(r2w1_tma<true, 2, 4>, "2r_1w_tma_bulk_U2_S4_x3", 2, 4, 3, true);
        tma(r2w1_tma<false, 1, 4>, "2r_1w_tma_stg_U1_S4_x6", 1, 4, 6, false);
        tma(r2w1_tma<true, 1, 4>, "2r_1w_tma_bulk_U1_S4_x6", 1, 4, 6, true);
        cudaError_t err = cudaGetLastError();
        if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
        return 0;
    }
    run("read_only", [&] { readonly<<<grid, block>>>(a, n, sink); }, (double)bytes);
    run("write_only", [&] { mix<<<grid, block>>>(a, b, 0, 1, n); }, (double)bytes);
    run("copy_1r_1w", [&] { mix<<<grid, block>>>(a, b, n, 1, n); }, 2.0 * bytes);
    run("1r_2w", [&] { mix<<<grid, block>>>(a, b, n / 2, 2, n); }, 1.5 * bytes);
    run("1r_6w", [&] { mix<<<grid, block>>>(a, b, n / 6, 6, n / 6 * 6); }, (double)bytes * 7 / 6);
    run("2r_1w", [&] { r2w1<<<grid, block>>>(a, b, n / 2); }, 1.5 * bytes);
    run("1r_6w_chunked", [&] { fanout_chunked<6><<<grid, block>>>(a, b, n / 6); }, (double)bytes * 7 / 6);
    cudaFuncSetAttribute(fanout_tma<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    run("1r_6w_tma", [&] { fanout_tma<6><<<2 * 148, block, 64 * 1024>>>(a, b, n / 6); }, (double)bytes * 7 / 6);
    run("1r_6w_tma_3cta", [&] { fanout_tma<6><<<3 * 148, block, 64 * 1024>>>(a, b, n / 6); }, (double)bytes * 7 / 6);
    cudaFuncSetAttribute(fanout_tma<6, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(fanout_tma<6, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    run("1r_6w_tma_8KB_2cta", [&] { fanout_tma<6, 2><<<2 * 148, block, 64 * 1024>>>(a, b, n / 6); }, (double)bytes * 7 / 6);
    run("1r_6w_tma_8KB_3cta", [&] { fanout_tma<6, 2><<<3 * 148, block, 64 * 1024>>>(a, b, n / 6); }, (double)bytes * 7 / 6);
    run("1r_6w_tma_16KB_3cta", [&] { fanout_tma<6, 4><<<3 * 148, block, 64 * 1024>>>(a, b, n / 6); }, (double)bytes * 7 / 6);
    run("1r_6w_tma_8KB_6cta", [&] { fanout_tma<6, 2><<<6 * 148, block, 32 * 1024>>>(a, b, n / 6); }, (double)bytes * 7 / 6);
    run("copy_ilp4", [&] { fanout_ilp<1, 4><<<grid, block>>>(a, b, n); }, 2.0 * bytes);
    run("copy_ilp8", [&] { fanout_ilp<1, 8><<<grid, block>>>(a, b, n); }, 2.0 * bytes);
    run("1r_2w_ilp4", [&] { fanout_ilp<2, 4><<<grid, block>>>(a, b, n / 2); }, 1.5 * bytes);
    run("1r_2w_ilp8", [&] { fanout_ilp<2, 8><<<grid, block>>>(a, b, n / 2); }, 1.5 * bytes);
    run("1r_2w_ilp8_2x", [&] { fanout_ilp<2, 8><<<2 * grid, block>>>(a, b, n / 2); }, 1.5 * bytes);
    cudaFuncSetAttribute(fanout_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(fanout_tma<2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    run("1r_2w_tma_2cta", [&] { fanout_tma<2><<<2 * 148, block, 64 * 1024>>>(a, b, n / 2); }, 1.5 * bytes);
    run("1r_2w_tma_3cta", [&] { fanout_tma<2><<<3 * 148, block, 64 * 1024>>>(a, b, n / 2); }, 1.5 * bytes);
    run("1r_2w_tma_16KB_3cta", [&] { fanout_tma<2, 4><<<3 * 148, block, 64 * 1024>>>(a, b, n / 2); }, 1.5 * bytes);
    run("1r_2w_warp_stg_16w", [&] { warp_rows<2, false><<<2 * 148, block>>>(a, b, n / 2); }, 1.5 * bytes);
    run("1r_2w_warp_bulk_16w", [&] { warp_rows<2, true><<<2 * 148, block>>>(a, b, n / 2); }, 1.5 * bytes);
    run("1r_6w_warp_stg_16w", [&] { warp_rows<6, false><<<2 * 148, block>>>(a, b, n / 6); }, (double)bytes * 7 / 6);
    run("1r_6w_warp_bulk_16w", [&] { warp_rows<6, true><<<2 * 148, block>>>(a, b, n / 6); }, (double)bytes * 7 / 6);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
    return 0;
}
