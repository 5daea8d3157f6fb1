// rt_dist.cu -- multi-GPU frame assembly behind rt_dist_init.
//
// PAPER.md:48 (§3, Fig. 1) divides the picture into N identical parts, one per processor, and
// PAPER.md:56 (§3, Fig. 2) makes the left/right channels the first level of parallelism.  Here
// one process drives each GPU of one node; every rank holds the same scene and camera and renders
// its tiles of each frame (rt_shard_tiles: world 2 = one eye per rank).  Rank 0's framebuffers
// receive the whole frame:
//
//   peer transport (default): rank 0 publishes, per frame, the CUDA IPC handles of its output
//     framebuffers in a host shared-memory ring; every other rank maps them (cached) and its
//     trace kernel's pack epilogue stores each finished pixel straight into rank 0's
//     framebuffers over NVLink (same-device IPC on a one-GPU box).  Ordering is device-side:
//     rank 0's stream posts "frame k started" (its framebuffers are free) before its own tiles,
//     each peer's stream waits for that post, renders, fences system-wide and posts "rank r done
//     with frame k" into rank 0's memory; rank 0's stream waits for every post before anything
//     enqueued after the frame.  No gather call, no unpack, no staging copy, no host barrier.
//   NCCL transport (RT_DIST_NCCL, or when peer mappings fail): each rank packs its tiles into a
//     shard buffer, ncclGather (group send/recv on older NCCL) collects them on rank 0 and
//     k_unpack_shards scatters them into the framebuffers.  libnccl.so.2 is loaded with dlopen,
//     so the library itself has no NCCL link dependency.
//
// Waits on the device are bounded (RT_DIST_TIMEOUT_S, default 60 s): a rank that never posts turns
// into RT_ERR_PEER on the next call instead of a hung GPU.
#include <dlfcn.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <cuda.h>

#include "rt_context.h"

namespace {

constexpr int DIST_SLOTS = 16;        // frames a rank may run ahead of another (descriptor ring)
constexpr int DIST_MAX_WORLD = 64;
constexpr uint32_t SHM_MAGIC = 0x52544232u;
constexpr int NCCL_RING = 4;          // shard / gather buffers in flight (NCCL transport)

// one frame's output framebuffers on rank 0, as published for the peers
struct FrameDesc {
    uint64_t seq;                     // frame number (written last, release; read first, acquire)
    unsigned char handle[2][64];      // cudaIpcMemHandle_t of the allocation holding each eye's FB
    uint64_t offset[2], pitch[2];
    uint32_t fmt[2], has[2];
    uint32_t W, H, depth, pad;
};

// host shared memory of one job (POSIX shm, named after the job id)
struct ShmBlock {
    uint32_t magic;
    int32_t world, transport, pad;
    unsigned char flags_handle[64];   // IPC handle of rank 0's DevFlags
    int32_t joined[DIST_MAX_WORLD];   // 1 + (peer mapping ok)
    int32_t left[DIST_MAX_WORLD];
    uint64_t consumed[DIST_MAX_WORLD];// last descriptor each rank has read
    FrameDesc desc[DIST_SLOTS];
};

// device flags in rank 0's memory (IPC-exported): start[s] = last frame rank 0 started in ring
// slot s; done[r][s] = last frame rank r finished in ring slot s
struct DevFlags {
    unsigned long long start[DIST_SLOTS];
    unsigned long long done[DIST_MAX_WORLD][DIST_SLOTS];
};

// ---------------------------------------------------------------- NCCL, loaded at run time
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[RT_DIST_ID_BYTES]; } ncclUniqueId;
enum { ncclSuccess_ = 0, ncclUint8_ = 1 };
struct Nccl {
    bool ok = false;
    int (*GetUniqueId)(ncclUniqueId*) = nullptr;
    int (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    int (*CommDestroy)(ncclComm_t) = nullptr;
    int (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*Gather)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;   // NCCL >= 2.28
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    const char* (*ErrStr)(int) = nullptr;
};

Nccl& nccl() {
    static Nccl n = [] {
        Nccl x;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return x;
        auto sym = [&](const char* s) { return dlsym(h, s); };
        x.GetUniqueId = reinterpret_cast<decltype(x.GetUniqueId)>(sym("ncclGetUniqueId"));
        x.CommInitRank = reinterpret_cast<decltype(x.CommInitRank)>(sym("ncclCommInitRank"));
        x.CommDestroy = reinterpret_cast<decltype(x.CommDestroy)>(sym("ncclCommDestroy"));
        x.Send = reinterpret_cast<decltype(x.Send)>(sym("ncclSend"));
        x.Recv = reinterpret_cast<decltype(x.Recv)>(sym("ncclRecv"));
        x.Gather = reinterpret_cast<decltype(x.Gather)>(sym("ncclGather"));
        x.GroupStart = reinterpret_cast<decltype(x.GroupStart)>(sym("ncclGroupStart"));
        x.GroupEnd = reinterpret_cast<decltype(x.GroupEnd)>(sym("ncclGroupEnd"));
        x.ErrStr = reinterpret_cast<decltype(x.ErrStr)>(sym("ncclGetErrorString"));
        x.ok = x.GetUniqueId && x.CommInitRank && x.CommDestroy && x.Send && x.Recv && x.GroupStart && x.GroupEnd &&
               x.ErrStr;
        return x;
    }();
    return n;
}

// ---------------------------------------------------------------- device-side ordering
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// rank 0: "frame seq started in this slot: its framebuffers are free"
__global__ void k_dist_post(unsigned long long* word, unsigned long long seq) { st_release_sys(word, seq); }

// a peer: its pixels of frame seq are in rank 0's framebuffers (the render kernel fenced
// system-wide at exit; the release store orders this post after every one of them)
__global__ void k_dist_signal(unsigned long long* word, unsigned long long seq) {
    __threadfence_system();
    st_release_sys(word, seq);
}

// wait until words[i * stride] >= seq for i in [0, n), i != skip; one warp, bounded by timeout
__global__ void k_dist_wait(const unsigned long long* words, int stride, int n, int skip, unsigned long long seq,
                            int* err, unsigned long long timeout_ns) {
    const unsigned long long t0 = global_ns();
    for (int i = threadIdx.x; i < n; i += 32) {
        if (i == skip) continue;
        while (ld_acquire_sys(words + (size_t)i * stride) < seq) {
            if (global_ns() - t0 > timeout_ns) {
                atomicExch(err, 1);
                return;
            }
            __nanosleep(200);
        }
    }
}

double timeout_s() {
    const char* e = getenv("RT_DIST_TIMEOUT_S");
    const double v = e ? atof(e) : 60.0;
    return v > 0 ? v : 60.0;
}

// host spin-wait with backoff; false on timeout
template <typename Pred>
bool host_wait(Pred pred, double limit_s) {
    const auto t0 = std::chrono::steady_clock::now();
    for (int it = 0;; ++it) {
        if (pred()) return true;
        if (it < 64) continue;
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit_s) return false;
        if (it < 1024) std::this_thread::yield();
        else std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

std::string shm_name_of(const unsigned char* id) {
    uint64_t h = 1469598103934665603ull;               // FNV-1a over the 128-byte job id
    for (int i = 0; i < RT_DIST_ID_BYTES; ++i) h = (h ^ id[i]) * 1099511628211ull;
    char b[40];
    snprintf(b, sizeof b, "/rtb200_%016llx", (unsigned long long)h);
    return b;
}

}  // namespace

struct DistState {
    int rank = 0, world = 1, transport = RT_DIST_PEER;
    std::string shm_name;
    ShmBlock* shm = nullptr;
    DevFlags* flags_local = nullptr;      // rank 0
    DevFlags* flags_remote = nullptr;     // ranks != 0: rank 0's flags, IPC-mapped
    int* h_err = nullptr;                 // device-wait timeout flag (mapped pinned host word)
    int* d_err = nullptr;
    uint64_t seq = 0;
    double timeout = 60.0;
    // completion of the last frame that used each ring slot on this rank: a frame reusing the slot
    // waits for it on the device, so a slot's flag words only ever move frame by frame, in order,
    // even with frames in flight on streams that complete out of order
    cudaEvent_t slot_ev[DIST_SLOTS] = {};
    bool slot_used[DIST_SLOTS] = {};
    struct Map {
        std::string key;
        void* ptr;
    };
    std::vector<Map> maps;                // rank 0 framebuffer allocations mapped by a peer
    // NCCL transport
    ncclComm_t comm = nullptr;
    void* shard[NCCL_RING] = {};
    void* gathered[NCCL_RING] = {};
    cudaEvent_t ring_ev[NCCL_RING] = {};
    bool ring_used[NCCL_RING] = {};
    uint64_t shard_bytes = 0;
};

namespace {

rt_status nccl_fail(int r, const char* what) {
    return rtb_fail(RT_ERR_PEER, "%s: %s", what, nccl().ErrStr ? nccl().ErrStr(r) : "NCCL error");
}

void unmap_all(DistState* D) {
    for (auto& m : D->maps) cudaIpcCloseMemHandle(m.ptr);
    D->maps.clear();
}

void free_state(DistState* D, bool unlink_shm) {
    if (!D) return;
    unmap_all(D);
    if (D->flags_remote) cudaIpcCloseMemHandle(D->flags_remote);
    if (D->flags_local) cudaFree(D->flags_local);
    if (D->comm && nccl().ok) nccl().CommDestroy(D->comm);
    for (int i = 0; i < NCCL_RING; ++i) {
        if (D->shard[i]) cudaFree(D->shard[i]);
        if (D->gathered[i]) cudaFree(D->gathered[i]);
        if (D->ring_ev[i]) cudaEventDestroy(D->ring_ev[i]);
    }
    for (auto& ev : D->slot_ev)
        if (ev) cudaEventDestroy(ev);
    if (D->h_err) cudaFreeHost(D->h_err);
    if (D->shm) munmap(D->shm, sizeof(ShmBlock));
    if (unlink_shm && !D->shm_name.empty()) shm_unlink(D->shm_name.c_str());
    delete D;
}

// the allocation holding dev_ptr: IPC handle of its base + the byte offset of dev_ptr in it
rt_status ipc_handle_of(const void* dev_ptr, unsigned char* handle, uint64_t* offset) {
    using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static void* fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess) f = nullptr;
        return f;
    }();
    if (!fn) return rtb_fail(RT_ERR_PEER, "cuMemGetAddressRange entry point unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (reinterpret_cast<GetRange>(fn)(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS)
        return rtb_fail(RT_ERR_PEER, "cuMemGetAddressRange failed for the framebuffer");
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) return rtb_fail(RT_ERR_PEER, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    memcpy(handle, &h, 64);
    *offset = (uint64_t)((CUdeviceptr)dev_ptr - base);
    return RT_OK;
}

rt_status map_handle(DistState* D, const unsigned char* handle, void** ptr) {
    const std::string key(reinterpret_cast<const char*>(handle), 64);
    for (auto& m : D->maps)
        if (m.key == key) {
            *ptr = m.ptr;
            return RT_OK;
        }
    if (D->maps.size() >= 64) {                     // bounded cache: drop the oldest mapping
        // frames in flight may still store through it: drain this rank's device work first
        // (rare: only a caller cycling through more than 64 distinct framebuffer allocations)
        const cudaError_t se = cudaDeviceSynchronize();
        if (se != cudaSuccess) return rtb_fail(RT_ERR_CUDA, "draining before unmapping a framebuffer: %s", cudaGetErrorString(se));
        cudaIpcCloseMemHandle(D->maps.front().ptr);
        D->maps.erase(D->maps.begin());
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    const cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return rtb_fail(RT_ERR_PEER, "cudaIpcOpenMemHandle (rank 0 framebuffer): %s", cudaGetErrorString(e));
    D->maps.push_back({key, *ptr});
    return RT_OK;
}

rt_status check_err(DistState* D) {
    if (D->h_err && __atomic_load_n(D->h_err, __ATOMIC_ACQUIRE))
        return rtb_fail(RT_ERR_PEER, "multi-GPU frame: a rank did not post within %.0f s (RT_DIST_TIMEOUT_S)", D->timeout);
    return RT_OK;
}

// ---------------------------------------------------------------- host protocol (shared memory)
// Create (rank 0) or attach to the job's shared block; rank 0 fills it (flags handle, world,
// transport) and sets the magic last.
rt_status shm_attach(DistState* D, uint32_t transport, const unsigned char* flags_handle) {
    int fd = -1;
    if (D->rank == 0) {
        shm_unlink(D->shm_name.c_str());            // a stale block of a crashed run with the same id
        fd = shm_open(D->shm_name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
        if (fd >= 0 && ftruncate(fd, sizeof(ShmBlock)) != 0) {
            close(fd);
            fd = -1;
        }
    } else {
        // open only once rank 0 has sized the block: between its shm_open and ftruncate the object
        // is 0 bytes, and touching a mapping past the end of the object raises SIGBUS
        host_wait([&] {
            if ((fd = shm_open(D->shm_name.c_str(), O_RDWR, 0600)) < 0) return false;
            struct stat sb;
            if (fstat(fd, &sb) == 0 && sb.st_size >= (off_t)sizeof(ShmBlock)) return true;
            close(fd);
            fd = -1;
            return false;
        }, D->timeout);
    }
    if (fd < 0) return rtb_fail(RT_ERR_PEER, "rt_dist_init: shared memory %s unavailable", D->shm_name.c_str());
    void* m = mmap(nullptr, sizeof(ShmBlock), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (m == MAP_FAILED) return rtb_fail(RT_ERR_PEER, "rt_dist_init: mmap of %s failed", D->shm_name.c_str());
    D->shm = static_cast<ShmBlock*>(m);
    ShmBlock* S = D->shm;
    if (D->rank == 0) {
        if (flags_handle) memcpy(S->flags_handle, flags_handle, 64);
        S->world = D->world;
        S->transport = (int32_t)transport;
        __atomic_store_n(&S->magic, SHM_MAGIC, __ATOMIC_RELEASE);
    } else if (!host_wait([&] { return __atomic_load_n(&S->magic, __ATOMIC_ACQUIRE) == SHM_MAGIC; }, D->timeout)) {
        return rtb_fail(RT_ERR_PEER, "rt_dist_init: rank 0 never initialised %s", D->shm_name.c_str());
    }
    if (S->world != D->world)
        return rtb_fail(RT_ERR_INVALID_ARG, "rt_dist_init: world %d, rank 0 says %d", D->world, S->world);
    return RT_OK;
}

// announce this rank (state 1 + ipc_ok) and wait until every rank has
rt_status shm_join(DistState* D, int ipc_ok) {
    ShmBlock* S = D->shm;
    __atomic_store_n(&S->joined[D->rank], 1 + ipc_ok, __ATOMIC_RELEASE);
    if (!host_wait([&] {
            for (int r = 0; r < D->world; ++r)
                if (!__atomic_load_n(&S->joined[r], __ATOMIC_ACQUIRE)) return false;
            return true;
        }, D->timeout))
        return rtb_fail(RT_ERR_PEER, "rt_dist_init: not every rank of %d joined within %.0f s", D->world, D->timeout);
    return RT_OK;
}

// rank 0: publish frame k's descriptor in ring slot k mod DIST_SLOTS, once every other rank has
// read the slot's previous frame (k - DIST_SLOTS)
rt_status ring_publish(DistState* D, uint64_t k, const FrameDesc& f) {
    ShmBlock* S = D->shm;
    const bool ok = host_wait([&] {
        for (int r = 1; r < D->world; ++r)
            if (__atomic_load_n(&S->consumed[r], __ATOMIC_ACQUIRE) + DIST_SLOTS < k) return false;
        return true;
    }, D->timeout);
    if (!ok) return rtb_fail(RT_ERR_PEER, "distributed frame %llu: a rank fell %d frames behind", (unsigned long long)k,
                             DIST_SLOTS);
    FrameDesc& d = S->desc[k % DIST_SLOTS];
    const uint64_t keep = d.seq;
    memcpy(&d, &f, sizeof d);
    d.seq = keep;
    __atomic_store_n(&d.seq, k, __ATOMIC_RELEASE);
    return RT_OK;
}

// ranks != 0: read frame k's descriptor and mark it consumed
rt_status ring_fetch(DistState* D, uint64_t k, FrameDesc* out) {
    ShmBlock* S = D->shm;
    FrameDesc& f = S->desc[k % DIST_SLOTS];
    if (!host_wait([&] { return __atomic_load_n(&f.seq, __ATOMIC_ACQUIRE) == k; }, D->timeout))
        return rtb_fail(RT_ERR_PEER, "distributed frame %llu: rank 0 did not publish it", (unsigned long long)k);
    memcpy(out, &f, sizeof *out);
    __atomic_store_n(&S->consumed[D->rank], k, __ATOMIC_RELEASE);
    return RT_OK;
}

// announce leaving; rank 0 waits for every rank (their mappings of its memory are closed)
bool shm_leave(DistState* D) {
    ShmBlock* S = D->shm;
    __atomic_store_n(&S->left[D->rank], 1, __ATOMIC_RELEASE);
    if (D->rank != 0) return true;
    return host_wait([&] {
        for (int r = 0; r < D->world; ++r)
            if (!__atomic_load_n(&S->left[r], __ATOMIC_ACQUIRE)) return false;
        return true;
    }, D->timeout);
}

}  // namespace

// ------------------------------------------------------------------------------ frames
static rt_status dist_frame(rt_context* c, DistState* D, const rt_render_params* p, const rt_outputs* out,
                            cudaStream_t stream, uint64_t k, int slot);

rt_status rtb_dist_render(rt_context* c, const rt_render_params* p, const rt_outputs* out, cudaStream_t stream) {
    DistState* D = c->dist;
    // an explicit tile subset (shard_world > 1) is a local render of those tiles, not a frame
    // (a one-rank world renders locally, except under an explicit RT_DIST_NCCL: then the frame goes
    // through the NCCL transport -- pack, a one-rank ncclGather, unpack -- the whole data path of a
    // multi-GPU frame, exercisable on one GPU)
    if (p->shard_world != 1 || (D->world == 1 && !D->comm)) return rtb_render_local(c, p, out, stream);
    rt_status st;
    if ((st = check_err(D))) return st;
    if (p->flags & ~(RT_RENDER_COUNT | RT_RENDER_BRUTE_FORCE | RT_RENDER_KDTREE))
        return rtb_fail(RT_ERR_INVALID_ARG, "distributed frame: flags 0x%x", p->flags);
    if (out->prim_id || out->radiance || out->shard || out->composed.dev_ptr)
        return rtb_fail(RT_ERR_INVALID_ARG, "distributed frame: framebuffer outputs only (ID / radiance / shard "
                                            "planes need an explicit shard render)");
    if (!c->has_scene) return rtb_fail(RT_ERR_NO_SCENE, "render before rt_scene_upload");
    if (!c->has_camera) return rtb_fail(RT_ERR_NO_CAMERA, "render before rt_set_stereo_camera");
    CUDA_TRY(cudaSetDevice(c->device));
    const uint64_t k = ++D->seq;
    const int slot = (int)(k % DIST_SLOTS);
    if (D->slot_used[slot]) CUDA_TRY(cudaStreamWaitEvent(stream, D->slot_ev[slot], 0));
    st = dist_frame(c, D, p, out, stream, k, slot);
    if (st) return st;
    CUDA_TRY(cudaEventRecord(D->slot_ev[slot], stream));
    D->slot_used[slot] = true;
    return RT_OK;
}

// frame k of a distributed context in ring slot `slot` (peer or NCCL transport)
static rt_status dist_frame(rt_context* c, DistState* D, const rt_render_params* p, const rt_outputs* out,
                            cudaStream_t stream, uint64_t k, int slot) {
    rt_status st;
    rt_render_params q = *p;
    q.shard_rank = (uint32_t)D->rank;
    q.shard_world = (uint32_t)D->world;
    const unsigned long long tmo = (unsigned long long)(D->timeout * 1e9);

    if (D->transport == RT_DIST_PEER) {
        if (D->rank == 0) {
            FrameDesc f{};
            const rt_fb fb[2] = {out->left, out->right};
            for (int e = 0; e < 2; ++e) {
                f.has[e] = fb[e].dev_ptr != nullptr;
                f.fmt[e] = fb[e].format;
                f.pitch[e] = fb[e].pitch_bytes;
                if (f.has[e] && (st = ipc_handle_of(fb[e].dev_ptr, f.handle[e], &f.offset[e]))) return st;
            }
            f.W = p->width;
            f.H = p->height;
            f.depth = p->max_depth;
            if ((st = ring_publish(D, k, f))) return st;
            k_dist_post<<<1, 1, 0, stream>>>(&D->flags_local->start[slot], k);
            CUDA_TRY(cudaGetLastError());
            if ((st = rtb_render_local(c, &q, out, stream))) return st;
            k_dist_wait<<<1, 32, 0, stream>>>(&D->flags_local->done[0][slot], DIST_SLOTS, D->world, 0, k, D->d_err, tmo);
            CUDA_TRY(cudaGetLastError());
            return RT_OK;
        }
        FrameDesc d;
        if ((st = ring_fetch(D, k, &d))) return st;
        if (d.W != p->width || d.H != p->height || d.depth != p->max_depth)
            return rtb_fail(RT_ERR_INVALID_ARG, "distributed frame %llu: rank 0 renders %ux%u depth %u, this rank %ux%u "
                                                "depth %u", (unsigned long long)k, d.W, d.H, d.depth, p->width,
                            p->height, p->max_depth);
        rt_outputs o{};
        rt_fb* fb[2] = {&o.left, &o.right};
        for (int e = 0; e < 2; ++e) {
            if (!d.has[e]) continue;
            void* base = nullptr;
            if ((st = map_handle(D, d.handle[e], &base))) return st;
            fb[e]->dev_ptr = static_cast<char*>(base) + d.offset[e];
            fb[e]->format = d.fmt[e];
            fb[e]->pitch_bytes = d.pitch[e];
        }
        o.counters = out->counters;
        q.flags |= RT_RENDER_PEER_STORE;
        k_dist_wait<<<1, 32, 0, stream>>>(&D->flags_remote->start[slot], 1, 1, -1, k, D->d_err, tmo);
        CUDA_TRY(cudaGetLastError());
        if ((st = rtb_render_local(c, &q, &o, stream))) return st;
        k_dist_signal<<<1, 1, 0, stream>>>(&D->flags_remote->done[D->rank][slot], k);
        CUDA_TRY(cudaGetLastError());
        return RT_OK;
    }

    // ---- NCCL transport: pack -> gather -> unpack
    const uint32_t fmt = out->left.dev_ptr ? out->left.format : out->right.format;
    if (D->rank == 0 && !out->left.dev_ptr && !out->right.dev_ptr)
        return rtb_fail(RT_ERR_INVALID_ARG, "distributed frame: rank 0 needs a framebuffer");
    uint64_t per = 0;
    if ((st = rt_shard_bytes(p->width, p->height, (uint32_t)D->world, RT_FORMAT_RGBA16F, &per))) return st;
    if (per > D->shard_bytes) {                     // grow the ring (sized for the wider format)
        CUDA_TRY(cudaDeviceSynchronize());
        for (int i = 0; i < NCCL_RING; ++i) {
            if (D->shard[i]) cudaFree(D->shard[i]);
            if (D->gathered[i]) cudaFree(D->gathered[i]);
            D->shard[i] = D->gathered[i] = nullptr;
            D->ring_used[i] = false;
            CUDA_TRY(cudaMalloc(&D->shard[i], per));
            if (D->rank == 0) CUDA_TRY(cudaMalloc(&D->gathered[i], per * D->world));
        }
        D->shard_bytes = per;
    }
    if ((st = rt_shard_bytes(p->width, p->height, (uint32_t)D->world, fmt, &per))) return st;
    const int r = (int)(k % NCCL_RING);
    if (D->ring_used[r]) CUDA_TRY(cudaStreamWaitEvent(stream, D->ring_ev[r], 0));
    rt_outputs o{};
    o.shard = D->shard[r];
    o.shard_format = fmt;
    o.counters = out->counters;
    if ((st = rtb_render_local(c, &q, &o, stream))) return st;
    Nccl& N = nccl();
    int res;
    if (N.Gather) {
        res = N.Gather(D->shard[r], D->gathered[r], per, ncclUint8_, 0, D->comm, stream);
        if (res != ncclSuccess_) return nccl_fail(res, "ncclGather");
    } else {
        if ((res = N.GroupStart()) != ncclSuccess_) return nccl_fail(res, "ncclGroupStart");
        if (D->rank == 0) {
            CUDA_TRY(cudaMemcpyAsync(D->gathered[r], D->shard[r], per, cudaMemcpyDeviceToDevice, stream));
            for (int src = 1; src < D->world && res == ncclSuccess_; ++src)
                res = N.Recv(static_cast<char*>(D->gathered[r]) + (size_t)src * per, per, ncclUint8_, src, D->comm, stream);
        } else {
            res = N.Send(D->shard[r], per, ncclUint8_, 0, D->comm, stream);
        }
        const int r2 = N.GroupEnd();
        if (res != ncclSuccess_) return nccl_fail(res, "ncclSend/ncclRecv");
        if (r2 != ncclSuccess_) return nccl_fail(r2, "ncclGroupEnd");
    }
    if (D->rank == 0 && (st = rtb_unpack_on(c, D->gathered[r], p->width, p->height, (uint32_t)D->world, fmt, out->left,
                                            out->right, stream)))
        return st;
    CUDA_TRY(cudaEventRecord(D->ring_ev[r], stream));
    D->ring_used[r] = true;
    return RT_OK;
}

void rtb_dist_destroy(rt_context* c) {
    if (!c->dist) return;
    free_state(c->dist, c->dist->rank == 0);
    c->dist = nullptr;
}

// ------------------------------------------------------------------------------ C ABI
extern "C" {

rt_status rt_dist_unique_id(void* id) {
    if (!id) return rtb_fail(RT_ERR_INVALID_ARG, "rt_dist_unique_id: NULL");
    memset(id, 0, RT_DIST_ID_BYTES);
    Nccl& N = nccl();
    if (N.ok) {
        ncclUniqueId u;
        const int r = N.GetUniqueId(&u);
        if (r == ncclSuccess_) {
            memcpy(id, &u, RT_DIST_ID_BYTES);
            return RT_OK;
        }
    }
    // no NCCL: a random job id (names the host rendezvous; the NCCL transport is then unavailable)
    unsigned char* b = static_cast<unsigned char*>(id);
    const int fd = open("/dev/urandom", O_RDONLY);
    ssize_t got = fd >= 0 ? read(fd, b, RT_DIST_ID_BYTES) : -1;
    if (fd >= 0) close(fd);
    if (got != RT_DIST_ID_BYTES) {
        const uint64_t t = (uint64_t)std::chrono::steady_clock::now().time_since_epoch().count() ^ ((uint64_t)getpid() << 32);
        for (int i = 0; i < RT_DIST_ID_BYTES; ++i) b[i] = (unsigned char)(t >> (8 * (i % 8))) ^ (unsigned char)(i * 131);
    }
    b[0] |= 1;                                      // never all zero
    return RT_OK;
}

rt_status rt_dist_init(rt_context* c, int rank, int world, const void* id, uint32_t flags) {
    NvtxRange nvtx_("rt_dist_init");
    if (!c || !id) return rtb_fail(RT_ERR_INVALID_ARG, "rt_dist_init: NULL argument");
    if (world < 1 || world > DIST_MAX_WORLD || rank < 0 || rank >= world)
        return rtb_fail(RT_ERR_INVALID_ARG, "rt_dist_init: rank %d of world %d (max %d)", rank, world, DIST_MAX_WORLD);
    if (flags > RT_DIST_NCCL) return rtb_fail(RT_ERR_INVALID_ARG, "rt_dist_init: flags %u", flags);
    if (c->dist) return rtb_fail(RT_ERR_INVALID_ARG, "rt_dist_init: context already in a world (rt_dist_finalize first)");
    CUDA_TRY(cudaSetDevice(c->device));
    DistState* D = new (std::nothrow) DistState();
    if (!D) return rtb_fail(RT_ERR_OOM, "rt_dist_init: host allocation");
    D->rank = rank;
    D->world = world;
    D->timeout = timeout_s();
    D->shm_name = shm_name_of(static_cast<const unsigned char*>(id));
    auto bail = [&](rt_status s) {
        free_state(D, rank == 0);
        return s;
    };
    cudaError_t e = cudaHostAlloc(&D->h_err, sizeof(int), cudaHostAllocMapped);
    if (e == cudaSuccess) {
        *D->h_err = 0;
        e = cudaHostGetDevicePointer(&D->d_err, D->h_err, 0);
    }
    if (e != cudaSuccess) return bail(rtb_fail(RT_ERR_CUDA, "rt_dist_init: mapped error word: %s", cudaGetErrorString(e)));
    // ---- rank 0's device flags every peer posts into, then the host rendezvous
    unsigned char fh[64] = {0};
    if (rank == 0) {
        e = cudaMalloc(&D->flags_local, sizeof(DevFlags));
        if (e == cudaSuccess) e = cudaMemset(D->flags_local, 0, sizeof(DevFlags));
        cudaIpcMemHandle_t h;
        if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, D->flags_local);
        if (e != cudaSuccess) return bail(rtb_fail(RT_ERR_CUDA, "rt_dist_init: device flags: %s", cudaGetErrorString(e)));
        memcpy(fh, &h, 64);
    }
    rt_status st;
    if ((st = shm_attach(D, flags, fh))) return bail(st);
    ShmBlock* S = D->shm;
    // ---- peer transport: map rank 0's flags (the first peer mapping; failure -> NCCL)
    int ipc_ok = 1;
    if (rank != 0 && S->transport == RT_DIST_PEER) {
        cudaIpcMemHandle_t h;
        memcpy(&h, S->flags_handle, 64);
        void* p = nullptr;
        if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) {
            D->flags_remote = static_cast<DevFlags*>(p);
        } else {
            cudaGetLastError();
            ipc_ok = 0;
        }
    }
    if ((st = shm_join(D, ipc_ok))) return bail(st);
    for (int i = 0; i < DIST_SLOTS; ++i)
        if ((e = cudaEventCreateWithFlags(&D->slot_ev[i], cudaEventDisableTiming)) != cudaSuccess)
            return bail(rtb_fail(RT_ERR_CUDA, "rt_dist_init: %s", cudaGetErrorString(e)));
    bool all_ipc = true;
    for (int r = 0; r < world; ++r) all_ipc = all_ipc && S->joined[r] == 2;
    D->transport = (S->transport == RT_DIST_PEER && all_ipc) ? RT_DIST_PEER : RT_DIST_NCCL;
    if (D->transport == RT_DIST_NCCL && (world > 1 || flags == RT_DIST_NCCL)) {
        if (!nccl().ok) return bail(rtb_fail(RT_ERR_PEER, "rt_dist_init: peer mappings failed and libnccl.so.2 is unavailable"));
        ncclUniqueId u;
        memcpy(&u, id, RT_DIST_ID_BYTES);
        const int r = nccl().CommInitRank(&D->comm, world, u, rank);
        if (r != ncclSuccess_) return bail(nccl_fail(r, "ncclCommInitRank (the id must come from rt_dist_unique_id with NCCL)"));
        for (int i = 0; i < NCCL_RING; ++i)
            if ((e = cudaEventCreateWithFlags(&D->ring_ev[i], cudaEventDisableTiming)) != cudaSuccess)
                return bail(rtb_fail(RT_ERR_CUDA, "rt_dist_init: %s", cudaGetErrorString(e)));
    }
    c->dist = D;
    return RT_OK;
}

rt_status rt_dist_finalize(rt_context* c) {
    NvtxRange nvtx_("rt_dist_finalize");
    if (!c) return rtb_fail(RT_ERR_INVALID_ARG, "rt_dist_finalize: NULL context");
    DistState* D = c->dist;
    if (!D) return RT_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaDeviceSynchronize());              // every frame of this rank is complete
    const rt_status err = check_err(D);
    unmap_all(D);
    if (D->flags_remote) {
        cudaIpcCloseMemHandle(D->flags_remote);
        D->flags_remote = nullptr;
    }
    const bool ok = shm_leave(D);                   // peers close their mappings before rank 0 frees
    free_state(D, D->rank == 0);
    c->dist = nullptr;
    if (!ok) return rtb_fail(RT_ERR_PEER, "rt_dist_finalize: not every rank left within the timeout");
    return err;
}

rt_status rt_dist_host_selftest(int rank, int world, const void* id, uint32_t frames, uint64_t* checksum) {
    if (!id || !checksum) return rtb_fail(RT_ERR_INVALID_ARG, "rt_dist_host_selftest: NULL argument");
    if (world < 1 || world > DIST_MAX_WORLD || rank < 0 || rank >= world)
        return rtb_fail(RT_ERR_INVALID_ARG, "rt_dist_host_selftest: rank %d of world %d", rank, world);
    DistState* D = new (std::nothrow) DistState();
    if (!D) return rtb_fail(RT_ERR_OOM, "rt_dist_host_selftest: host allocation");
    D->rank = rank;
    D->world = world;
    D->timeout = timeout_s();
    D->shm_name = shm_name_of(static_cast<const unsigned char*>(id));
    rt_status st = shm_attach(D, RT_DIST_PEER, nullptr);
    if (!st) st = shm_join(D, 1);
    uint64_t h = 1469598103934665603ull;
    for (uint64_t k = 1; !st && k <= frames; ++k) {
        FrameDesc f{};
        if (rank == 0) {                            // synthetic descriptor of frame k
            f.W = (uint32_t)(k * 7 + 1);
            f.H = (uint32_t)(k * 13 + 2);
            f.depth = (uint32_t)(k % 17);
            f.offset[0] = k * 1000003ull;
            f.offset[1] = k * 999983ull;
            f.handle[0][k % 64] = (unsigned char)k;
            st = ring_publish(D, k, f);
        } else {
            st = ring_fetch(D, k, &f);
        }
        const uint64_t v[5] = {f.W, f.H, f.depth, f.offset[0] ^ f.offset[1], f.handle[0][k % 64]};
        for (uint64_t x : v) h = (h ^ x) * 1099511628211ull;
    }
    if (!st && !shm_leave(D)) st = rtb_fail(RT_ERR_PEER, "rt_dist_host_selftest: not every rank left");
    *checksum = h;
    free_state(D, rank == 0);
    return st;
}

rt_status rt_dist_info(rt_context* c, int32_t info[4]) {
    if (!c || !info) return rtb_fail(RT_ERR_INVALID_ARG, "rt_dist_info: NULL argument");
    const DistState* D = c->dist;
    info[0] = D ? D->rank : 0;
    info[1] = D ? D->world : 1;
    info[2] = D ? D->transport : -1;
    info[3] = D ? (int32_t)D->seq : 0;
    return RT_OK;
}

}  // extern "C"
