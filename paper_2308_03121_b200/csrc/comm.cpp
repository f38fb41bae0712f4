// comm.cpp -- the multi-GPU part of the C ABI (include/nnvisr.h "Multi-GPU
// frame-range shards"): shard geometry, the halo message plan, and the NCCL
// halo exchange over NVLink (SURVEY.md §8(b) nnvisr_comm_* / nnvisr_halo_exchange,
// §8(e)).
//
// Why an exchange at all (§3.3): a tuple near a shard edge
// reads up to L frames before the shard and N-1-L after it, and whether those
// frames are used or replaced by duplicates depends on their scene-cut flags
// (§3.2).  So each rank needs its neighbours' edge frames and
// flags: one grouped point-to-point exchange, nothing else crosses ranks.
//
// NCCL is loaded at run time (dlopen of libnccl.so.2; the copy torch already
// loaded is reused), so the library itself does not depend on NCCL: without
// it the nnvisr_comm_* calls return NNVISR_ERR_NCCL and everything else works.
#include "nnvisr.h"

#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

using namespace nnvisr;

struct nnvisr_comm {
    ncclComm_t comm;
    int32_t rank, world, device;
};

namespace {

// ------------------------------------------------------------- NCCL loading
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetVersion)(int *);
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*CommInitAll)(ncclComm_t *, int, const int *);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *);
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    const char *(*GetErrorString)(ncclResult_t);
};

NcclApi g_nccl;
std::once_flag g_nccl_once;

void load_nccl()
{
    void *lib = nullptr;
    const char *env = std::getenv("NNVISR_NCCL_LIB");
    if (env && *env) {
        lib = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    } else {
        lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // torch's copy, if loaded
        if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    }
    if (!lib) {
        const char *e = dlerror();
        g_nccl.why = std::string("cannot load NCCL (libnccl.so.2): ") + (e ? e : "?");
        return;
    }
#define NNVISR_SYM(name)                                                              \
    *reinterpret_cast<void **>(&g_nccl.name) = dlsym(lib, "nccl" #name);             \
    if (!g_nccl.name) {                                                               \
        g_nccl.why = "NCCL library lacks nccl" #name;                                 \
        return;                                                                       \
    }
    NNVISR_SYM(GetVersion)
    NNVISR_SYM(GetUniqueId)
    NNVISR_SYM(CommInitRank)
    NNVISR_SYM(CommInitAll)
    NNVISR_SYM(CommDestroy)
    NNVISR_SYM(CommGetAsyncError)
    NNVISR_SYM(Send)
    NNVISR_SYM(Recv)
    NNVISR_SYM(AllGather)
    NNVISR_SYM(GroupStart)
    NNVISR_SYM(GroupEnd)
    NNVISR_SYM(GetErrorString)
#undef NNVISR_SYM
    g_nccl.ok = true;
}

nnvisr_status need_nccl()
{
    std::call_once(g_nccl_once, load_nccl);
    if (!g_nccl.ok) return set_error(NNVISR_ERR_NCCL, g_nccl.why.c_str());
    return NNVISR_OK;
}

nnvisr_status nccl_fail(ncclResult_t r, const char *what)
{
    char buf[384];
    std::snprintf(buf, sizeof buf, "%s: %s (ncclResult %d)", what, g_nccl.GetErrorString(r), (int)r);
    return set_error(NNVISR_ERR_NCCL, buf);
}

nnvisr_status arg_fail(const char *what) { return set_error(NNVISR_ERR_INVALID_ARG, what); }

// Asynchronous errors of a communicator (a failed peer, a network error):
// ncclCommGetAsyncError after every grouped call and on request.
nnvisr_status check_async(const nnvisr_comm *c)
{
    ncclResult_t a = ncclSuccess;
    ncclResult_t r = g_nccl.CommGetAsyncError(c->comm, &a);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommGetAsyncError");
    if (a != ncclSuccess && a != ncclInProgress) return nccl_fail(a, "asynchronous NCCL error");
    return NNVISR_OK;
}

// Enqueue the frame and flag messages of one rank (inside a group).
nnvisr_status enqueue_rank(const nnvisr_comm *c, int64_t total, int32_t L, int32_t R, void *window,
                           int64_t frame_bytes, uint8_t *cut_window, cudaStream_t st)
{
    nnvisr_halo_msg msg[4];
    int32_t nm = 0;
    nnvisr_status s = nnvisr_halo_plan(total, c->world, c->rank, L, R, msg, &nm);
    if (s) return s;
    for (int i = 0; i < nm; ++i) {
        const nnvisr_halo_msg &m = msg[i];
        ncclResult_t r = ncclSuccess;
        if (window) {
            char *p = static_cast<char *>(window) + m.first * frame_bytes;
            const size_t n = static_cast<size_t>(m.count * frame_bytes);
            r = m.send ? g_nccl.Send(p, n, ncclUint8, m.peer, c->comm, st)
                       : g_nccl.Recv(p, n, ncclUint8, m.peer, c->comm, st);
            if (r != ncclSuccess) return nccl_fail(r, m.send ? "ncclSend (halo frames)" : "ncclRecv (halo frames)");
        }
        if (cut_window) {
            uint8_t *p = cut_window + m.first;
            r = m.send ? g_nccl.Send(p, (size_t)m.count, ncclUint8, m.peer, c->comm, st)
                       : g_nccl.Recv(p, (size_t)m.count, ncclUint8, m.peer, c->comm, st);
            if (r != ncclSuccess) return nccl_fail(r, m.send ? "ncclSend (halo flags)" : "ncclRecv (halo flags)");
        }
    }
    return NNVISR_OK;
}

nnvisr_status check_window(int64_t total, int32_t world, int32_t rank, int32_t L, int32_t R, void *window,
                           int64_t frame_bytes, uint8_t *cut_window)
{
    if (!window && !cut_window) return arg_fail("halo exchange: window and cut_window are both NULL");
    if (window && frame_bytes <= 0) return arg_fail("halo exchange: frame_bytes must be > 0");
    nnvisr_shard sh;
    return nnvisr_shard_of(total, world, rank, L, R, &sh);
}

}  // namespace

extern "C" {

nnvisr_status nnvisr_shard_of(int64_t total, int32_t world, int32_t rank, int32_t L, int32_t R, nnvisr_shard *out)
{
    if (!out) return arg_fail("nnvisr_shard_of: out is NULL");
    if (total < 0 || world < 1 || rank < 0 || rank >= world || L < 0 || R < 0 || L > 15 || R > 15)
        return arg_fail("nnvisr_shard_of: need total >= 0, 0 <= rank < world, 0 <= L, R <= 15");
    const int64_t a = (int64_t)rank * total / world, b = ((int64_t)rank + 1) * total / world;
    const int64_t need = L > R ? L : R;
    if (world > 1 && b - a < (need > 1 ? need : 1)) {
        char buf[160];
        std::snprintf(buf, sizeof buf, "shard %d of %d has %lld frames, fewer than the halo (L %d, R %d)", rank,
                      world, (long long)(b - a), L, R);
        return set_error(NNVISR_ERR_INVALID_ARG, buf);
    }
    out->begin = a;
    out->end = b;
    out->left = a < L ? a : L;
    out->right = total - b < R ? total - b : R;
    out->window_first = a - out->left;
    out->window_count = out->left + (b - a) + out->right;
    return NNVISR_OK;
}

nnvisr_status nnvisr_halo_plan(int64_t total, int32_t world, int32_t rank, int32_t L, int32_t R,
                               nnvisr_halo_msg msgs[4], int32_t *count)
{
    if (!msgs || !count) return arg_fail("nnvisr_halo_plan: NULL output");
    *count = 0;
    nnvisr_shard s;
    nnvisr_status st = nnvisr_shard_of(total, world, rank, L, R, &s);
    if (st) return st;
    const int64_t own0 = s.left, own1 = s.left + (s.end - s.begin);
    int32_t n = 0;
    if (rank > 0) {
        // rank-1's right halo = my first min(R, total - begin) frames
        const int64_t need = total - s.begin < R ? total - s.begin : R;
        if (need > 0) msgs[n++] = nnvisr_halo_msg{rank - 1, 1, own0, need};
        if (s.left > 0) msgs[n++] = nnvisr_halo_msg{rank - 1, 0, 0, s.left};
    }
    if (rank < world - 1) {
        // rank+1's left halo = my last min(L, end) frames
        const int64_t need = s.end < L ? s.end : L;
        if (need > 0) msgs[n++] = nnvisr_halo_msg{rank + 1, 1, own1 - need, need};
        if (s.right > 0) msgs[n++] = nnvisr_halo_msg{rank + 1, 0, own1, s.right};
    }
    *count = n;
    return NNVISR_OK;
}

nnvisr_status nnvisr_comm_unique_id(uint8_t id[NNVISR_COMM_ID_BYTES])
{
    if (!id) return arg_fail("nnvisr_comm_unique_id: id is NULL");
    nnvisr_status s = need_nccl();
    if (s) return s;
    ncclUniqueId u;
    ncclResult_t r = g_nccl.GetUniqueId(&u);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    static_assert(sizeof(u) == NNVISR_COMM_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id, &u, sizeof u);
    return NNVISR_OK;
}

nnvisr_status nnvisr_comm_init_rank(const uint8_t id[NNVISR_COMM_ID_BYTES], int32_t world, int32_t rank,
                                    nnvisr_comm **out)
{
    if (!id || !out) return arg_fail("nnvisr_comm_init_rank: NULL argument");
    if (world < 1 || rank < 0 || rank >= world) return arg_fail("nnvisr_comm_init_rank: need 0 <= rank < world");
    nnvisr_status s = need_nccl();
    if (s) return s;
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return set_error(NNVISR_ERR_CUDA, cudaGetErrorString(e));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    ncclComm_t c = nullptr;
    ncclResult_t r = g_nccl.CommInitRank(&c, world, u, rank);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
    *out = new nnvisr_comm{c, rank, world, dev};
    return NNVISR_OK;
}

nnvisr_status nnvisr_comm_init_all(int32_t ndev, const int32_t *devs, nnvisr_comm **comms)
{
    if (ndev < 1 || !devs || !comms) return arg_fail("nnvisr_comm_init_all: need ndev >= 1 and arrays");
    nnvisr_status s = need_nccl();
    if (s) return s;
    std::vector<ncclComm_t> c(ndev, nullptr);
    std::vector<int> d(devs, devs + ndev);
    ncclResult_t r = g_nccl.CommInitAll(c.data(), ndev, d.data());
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitAll");
    for (int i = 0; i < ndev; ++i) comms[i] = new nnvisr_comm{c[i], i, ndev, devs[i]};
    return NNVISR_OK;
}

nnvisr_status nnvisr_comm_info(const nnvisr_comm *comm, int32_t *rank, int32_t *world, int32_t *device)
{
    if (!comm) return arg_fail("nnvisr_comm_info: NULL communicator");
    if (rank) *rank = comm->rank;
    if (world) *world = comm->world;
    if (device) *device = comm->device;
    return NNVISR_OK;
}

nnvisr_status nnvisr_comm_check(const nnvisr_comm *comm)
{
    if (!comm) return arg_fail("nnvisr_comm_check: NULL communicator");
    nnvisr_status s = need_nccl();
    if (s) return s;
    return check_async(comm);
}

nnvisr_status nnvisr_halo_exchange(nnvisr_comm *comm, int64_t total_frames, int32_t L, int32_t R, void *window,
                                   int64_t frame_bytes, uint8_t *cut_window, void *stream)
{
    if (!comm) return arg_fail("nnvisr_halo_exchange: NULL communicator");
    nnvisr_status s = check_window(total_frames, comm->world, comm->rank, L, R, window, frame_bytes, cut_window);
    if (s) return s;
    if ((s = need_nccl())) return s;
    if (comm->world == 1) return check_async(comm);  // nothing crosses ranks
    ncclResult_t r = g_nccl.GroupStart();
    if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
    s = enqueue_rank(comm, total_frames, L, R, window, frame_bytes, cut_window, static_cast<cudaStream_t>(stream));
    r = g_nccl.GroupEnd();  // always close the group, even after a failed enqueue
    if (s) return s;
    if (r != ncclSuccess) return nccl_fail(r, "ncclGroupEnd");
    return check_async(comm);
}

nnvisr_status nnvisr_halo_exchange_all(nnvisr_comm *const *comms, int32_t ndev, int64_t total_frames, int32_t L,
                                       int32_t R, void *const *windows, int64_t frame_bytes,
                                       uint8_t *const *cut_windows, void *const *streams)
{
    if (ndev < 1 || !comms || !windows || !cut_windows || !streams)
        return arg_fail("nnvisr_halo_exchange_all: need ndev >= 1 and arrays");
    for (int i = 0; i < ndev; ++i) {
        if (!comms[i] || comms[i]->rank != i || comms[i]->world != ndev)
            return arg_fail("nnvisr_halo_exchange_all: comms must be the ndev ranks of one nnvisr_comm_init_all");
        nnvisr_status s = check_window(total_frames, ndev, i, L, R, windows[i], frame_bytes, cut_windows[i]);
        if (s) return s;
    }
    nnvisr_status s = need_nccl();
    if (s) return s;
    if (ndev > 1) {
        ncclResult_t r = g_nccl.GroupStart();
        if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
        for (int i = 0; i < ndev && !s; ++i)
            s = enqueue_rank(comms[i], total_frames, L, R, windows[i], frame_bytes, cut_windows[i],
                             static_cast<cudaStream_t>(streams[i]));
        r = g_nccl.GroupEnd();
        if (s) return s;
        if (r != ncclSuccess) return nccl_fail(r, "ncclGroupEnd");
    }
    for (int i = 0; i < ndev; ++i)
        if ((s = check_async(comms[i]))) return s;
    return NNVISR_OK;
}

nnvisr_status nnvisr_cut_allgather(nnvisr_comm *comm, int64_t *last_cuts, void *stream)
{
    if (!comm || !last_cuts) return arg_fail("nnvisr_cut_allgather: NULL argument");
    nnvisr_status s = need_nccl();
    if (s) return s;
    // in place: this rank's element is the send buffer (world 1: a no-op copy)
    ncclResult_t r = g_nccl.AllGather(last_cuts + comm->rank, last_cuts, 1, ncclInt64, comm->comm,
                                      static_cast<cudaStream_t>(stream));
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather (last scene cuts)");
    return check_async(comm);
}

nnvisr_status nnvisr_last_cut(const uint8_t *cut, int64_t first, int64_t count, int64_t *last_cut)
{
    if (!last_cut || (count > 0 && !cut) || first < 0 || count < 0) return arg_fail("nnvisr_last_cut: bad argument");
    *last_cut = -1;
    for (int64_t i = count - 1; i >= 0; --i)
        if (cut[i] && first + i > 0) {  // cut[0] of the clip is ignored (reading A9)
            *last_cut = first + i;
            break;
        }
    return NNVISR_OK;
}

nnvisr_status nnvisr_scene_start_scan(int32_t world, int32_t rank, const int64_t *last_cuts, int64_t begin,
                                      uint8_t cut_begin, int64_t *scene_start)
{
    if (!last_cuts || !scene_start || world < 1 || rank < 0 || rank >= world || begin < 0)
        return arg_fail("nnvisr_scene_start_scan: bad argument");
    // exclusive prefix max of the ranks' last cuts (every frame of ranks
    // j < rank lies before `begin`), unless `begin` itself starts a scene
    int64_t sc = 0;
    for (int32_t j = 0; j < rank; ++j) {
        if (last_cuts[j] >= begin) return arg_fail("nnvisr_scene_start_scan: a lower rank's cut lies at or after begin");
        sc = last_cuts[j] > sc ? last_cuts[j] : sc;
    }
    *scene_start = (cut_begin && begin > 0) ? begin : sc;
    return NNVISR_OK;
}

nnvisr_status nnvisr_comm_destroy(nnvisr_comm *comm)
{
    if (!comm) return NNVISR_OK;
    nnvisr_status s = need_nccl();
    if (s) return s;
    ncclResult_t r = g_nccl.CommDestroy(comm->comm);
    delete comm;
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
    return NNVISR_OK;
}

int32_t nnvisr_nccl_version(void)
{
    if (need_nccl()) return -1;
    int v = 0;
    if (g_nccl.GetVersion(&v) != ncclSuccess) return -1;
    return v;
}

}  // extern "C"
