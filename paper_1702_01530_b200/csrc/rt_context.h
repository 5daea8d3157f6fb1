// rt_context.h -- the library-private state behind an rt_context* (host runtime, rt_api.cu and
// rt_dist.cu) and the error / tracing helpers every entry point uses.
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/rt_b200.h"
#include "rt_internal.h"

// Sets the thread-local message returned by rt_last_error() and returns s.
rt_status rtb_fail(rt_status s, const char* fmt, ...);

#define CUDA_TRY(call)                                                                           \
    do {                                                                                         \
        cudaError_t e_ = (call);                                                                 \
        if (e_ != cudaSuccess) {                                                                 \
            if (e_ == cudaErrorMemoryAllocation)                                                 \
                return rtb_fail(RT_ERR_OOM, "%s: %s", #call, cudaGetErrorString(e_));            \
            return rtb_fail(RT_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_));               \
        }                                                                                        \
    } while (0)

// NVTX range over a C-ABI call (SURVEY §5 tracing): visible in Nsight Systems timelines, free
// when no tool is attached (NVTX3 is header-only)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

constexpr int RENDER_SLOTS = 16;

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
};

struct DistState;   // rt_dist.cu: multi-GPU frame assembly (rt_dist_init)

// device tile table of a block shard layout (RT_SHARD_BLOCK > 1), cached per layout
struct RtTileTable {
    uint32_t W = 0, H = 0, world = 0;
    int rank = 0, block = 1;    // rank -1: every rank's tiles (unpack)
    DevBuf buf;
};

struct rt_event {
    cudaEvent_t ev = nullptr;
};

struct rt_context {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t order_ev = nullptr;
    int num_sms = 148;
    int* work_counter = nullptr;    // [64]: 16 rotating render queues, 4 ints apart
    unsigned render_seq = 0;
    // completion event of the last render that used each work-queue slot: a render that reuses a
    // slot waits for it on the device (cudaStreamWaitEvent), and scene changes wait for all of them
    cudaEvent_t slot_ev[RENDER_SLOTS] = {};
    bool slot_used[RENDER_SLOTS] = {};
    // pinned staging of rt_scene_upload / rt_scene_update_vertices (grow-only)
    void* staging = nullptr;
    size_t staging_bytes = 0;
    unsigned long long* scratch_counters = nullptr;
    float* ffma_out = nullptr;
    // scene
    bool has_scene = false;
    std::vector<DevBuf> scene_bufs;
    rtb::DevScene sc{};
    uint64_t info[8] = {0};
    // camera
    bool has_camera = false;
    double cam_eye[2][3], cam_f[3], cam_r[3], cam_u[3], cam_th, cam_sigma_unit;
    float vfov = 0;
    int spec_mask = 7;               // scene-specialised trace instantiations allowed (bit 0 TRI, 1 OPAQUE, 2 LEAF1; env RT_SPEC_MASK, A/B only)
    int scene_leaf_max = 1;          // leaf_max of the uploaded scene's BVH (LEAF1 needs 1)
    int leaf_max = 1;                // LBVH leaf collapse threshold (env RT_LEAF_MAX, <= 16)
    int treelet_passes = 0;          // SAH treelet restructuring passes (env RT_TREELETS; 0 after a full
                                     // SAH build: measured neutral to slightly worse, DESIGN §5 r2)
    int sah_big = 4096;              // SAH tasks above this many items are split over many CTAs (env RT_SAH_BIG >= 2048)
    int sah_subtrees = 2;            // binned-SAH rebuild: 1 LBVH subtrees <= 16K prims, 2 the whole tree,
                                     // 0 off (env RT_SAH_SUBTREES)
    int collapse_dp = 1;             // SAH-optimal BVH4 collapse (env RT_COLLAPSE_DP=0: largest-area opening)
    float collapse_cprim = 0.4f;     // its primitive-test cost relative to a node visit (env RT_COLLAPSE_CPRIM)
    int grid_limit = 0;              // cap on trace CTAs (env RT_GRID_LIMIT; 0 = full machine)
    void* arena = nullptr;           // BVH build scratch (grow-only)
    size_t arena_bytes = 0;
    // refit state (rt_scene_update_vertices)
    int* d_prim_orig = nullptr;
    float* d_vertices = nullptr;
    uint32_t* d_tri = nullptr;
    float4* d_spheres = nullptr;
    uint32_t n_vertices = 0;
    std::vector<int> level_start;
    std::vector<uint32_t> h_tri;
    double sphere_bound = 0.0;
    struct IpcMap {
        std::string key;            // the 64-byte cudaIpcMemHandle_t
        void* ptr;
        int refs;
    };
    std::vector<IpcMap> ipc_maps;    // peer allocations mapped by rt_ipc_open (reference counted)
    // NEXT-4 kd-tree ablation (rt_kdtree_build)
    DevBuf kd_nodes_buf, kd_refs_buf;
    // multi-GPU frame assembly (rt_dist_init); null = single GPU
    DistState* dist = nullptr;
    std::vector<RtTileTable> tile_tables;
};

// Enqueue one render of params/outputs exactly as given (one GPU, no frame assembly); rt_api.cu.
rt_status rtb_render_local(rt_context* c, const rt_render_params* p, const rt_outputs* out, cudaStream_t stream);
// rt_dist.cu: a frame of a distributed context (this rank's tiles + assembly on rank 0), and teardown.
rt_status rtb_dist_render(rt_context* c, const rt_render_params* p, const rt_outputs* out, cudaStream_t stream);
void rtb_dist_destroy(rt_context* c);
// rt_unpack_shards on a given stream (rt_api.cu)
rt_status rtb_unpack_on(rt_context* c, const void* gathered, uint32_t W, uint32_t H, uint32_t world, uint32_t format,
                        rt_fb left, rt_fb right, cudaStream_t stream);
