// rt_internal.h -- shared between the host runtime (rt_api.cu) and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/rt_b200.h"
#include "rt_device.cuh"

enum {
    CNT_PRIMARY = RT_CNT_PRIMARY,
    CNT_REFLECTION = RT_CNT_REFLECTION,
    CNT_REFRACTION = RT_CNT_REFRACTION,
    CNT_SHADOW = RT_CNT_SHADOW,
    CNT_NODE_VISITS = RT_CNT_NODE_VISITS,
    CNT_TRI_TESTS = RT_CNT_TRI_TESTS,
    CNT_SPHERE_TESTS = RT_CNT_SPHERE_TESTS,
    CNT_PLANE_TESTS = RT_CNT_PLANE_TESTS,
    CNT_SHADE_HITS = RT_CNT_SHADE_HITS,
    CNT_LIGHT_EVALS = RT_CNT_LIGHT_EVALS,
    CNT_MISSES = RT_CNT_MISSES,
    CNT_PIXELS = RT_CNT_PIXELS,
    CNT_BOX_TESTS = RT_CNT_BOX_TESTS,
};
#define RT_NUM_COUNTERS_INTERNAL RT_NUM_COUNTERS

struct TraceParams {
    rtb::DevScene sc;
    rtb::DevCamera cam;
    int W, H, max_depth;
    int* work_counter;
    int n_work;             // work items (pixels incl. tile padding) of this shard
    int tiles_x, tiles_per_eye;
    int shard_mode;         // 0 one rank, 1 eye split (world 2), 2 tile pairs round-robin (world >= 3)
    int shard_rank, shard_world;
    const int* tile_list;   // mode 2 block layout: this rank's tile indices (null = round-robin tiles)
    void* fb[2];
    int fb_fmt[2];
    long long fb_pitch[2];
    int* prim_id;
    float4* radiance;
    void* shard;
    int shard_fmt;
    unsigned long long* counters;
    int stack_entries;      // BVH traversal stack depth (shared memory, [entry][thread])
    int n_tiles;            // 16x16 tiles in this shard (= n_work / 256)
    int peer_fence;         // framebuffers live in a peer's memory: fence system-wide at exit
    int fb_vec[2];          // rows 16-byte aligned (base and pitch): vectorised row stores
    void* comp;             // fused stereo composition output (RGBA8), null = none
    long long comp_pitch;
    int comp_mode;          // RT_COMPOSE_ANAGLYPH / RT_COMPOSE_SBS
    int comp_vec;           // composed rows 16-byte aligned
};

struct UnpackParams {
    void* left;
    void* right;
    long long pitch;
    int fmt;
    int W, H, tiles_x, tiles_per_eye, tiles_per_rank;
    int world, shard_mode;
    const int* gtile;       // block layout: [world][tiles_per_rank / 2] tile indices, -1 pad (null = round-robin)
};

// BVH build scratch (device pointers), owned by the context.
struct BuildBuffers {
    const float4* spheres;      // [S] (c, r)
    const float* vertices;      // [3V]
    const uint32_t* tri_idx;    // [3T]
    const uint32_t* tri_mat;    // [T]
    const uint32_t* sphere_mat; // [S]
    int n_spheres, n_planes, n_tris;
    float4* prims_unsorted;     // [3N]
    float4* prims;              // [3N] leaf order
    float4* aabb_lo;            // [N]
    float4* aabb_hi;            // [N]
    float4* centroid;           // [N]
    float4* leaf_lo;            // [N] leaf-order AABBs
    float4* leaf_hi;            // [N]
    unsigned int* bounds;       // [6] ordered-int centroid bounds
    uint32_t* keys[2];          // [N]
    uint32_t* vals[2];          // [N]
    uint32_t* hist;             // [256 * nblocks]
    int* left;                  // [N-1] child encodings
    int* right;                 // [N-1]
    int* parent_int;            // [N-1]
    int* parent_leaf;           // [N]
    int* flags;                 // [N-1]
    float4* node_lo;            // [N-1]
    float4* node_hi;            // [N-1]
    float4* nodes4;             // [7 * (N-1)] BVH4 nodes (upper bound; compacted by the caller)
    int2* frontier[2];          // [N] collapse work lists (bvh2 node, bvh4 slot)
    int* wide_counters;         // [2] next-frontier size, next BVH4 slot
    int2* range;                // [N-1] sorted primitive range of each internal node
    int* prim_orig;             // out: leaf slot -> original primitive index (kept for refit)
    int leaf_max;               // collapse subtrees of <= leaf_max primitives into leaves
    float* cost;                // [N-1] SAH cost of each internal node's subtree (treelets)
    int* count;                 // [N-1] primitives below each internal node (treelets)
    int treelet_passes;         // 0 = plain LBVH
    int sah_subtrees;           // binned SAH: 1 LBVH subtrees of <= 16384 primitives, 2 the whole tree
    int sah_big;                // SAH tasks above this many items run on many CTAs (chunked), others on a warp
    int collapse_dp;            // BVH2 -> BVH4 by the SAH-optimal DP (else largest-area-first opening)
    float collapse_cprim;       // DP cost of a primitive test relative to a BVH4 node visit
};

namespace rtb {
// NEXT-4 kd-tree ablation (rt_kdtree.cu): host-built binned-SAH kd-tree over the primitive records
struct KdHost {
    std::vector<int2> nodes;    // preorder; see rt_kdtree.cu for the encoding
    std::vector<int> refs;      // leaf reference lists (BVH primitive slots)
    int depth = 0, leaves = 0;
    float lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};   // root cell
};
void kd_build_host(const float4* prims, int n, int n_spheres, int max_leaf, int max_depth, KdHost& out);
}  // namespace rtb

// launchers (rt_trace.cu); flags = RT_RENDER_COUNT | _BRUTE_FORCE | _KDTREE, or RTB_TRACE_COMPOSE
// alone (the product kernel with the fused stereo composition in its epilogue)
constexpr unsigned RTB_TRACE_COMPOSE = 1u << 31;
constexpr unsigned RTB_TRACE_TRI = 1u << 30;       // the scene holds triangles only (product instantiation)
constexpr unsigned RTB_TRACE_OPAQUE = 1u << 29;    // no material refracts (product instantiation)
constexpr unsigned RTB_TRACE_LEAF1 = 1u << 28;     // every BVH leaf holds one primitive (product instantiation)
cudaError_t rtb_launch_trace(const TraceParams& P, unsigned flags, int grid, cudaStream_t st);
cudaError_t rtb_trace_occupancy(unsigned flags, int stack_entries, int* blocks_per_sm);
size_t rtb_trace_smem(int stack_entries);
int rtb_trace_block();      // threads per trace CTA (RT_BLOCK)
struct QueryParams {
    rtb::DevScene sc;
    const float* o;
    const float* d;
    const float* tmax;
    float* out_t;
    int* out_id;
    unsigned n;
    int any, brute;
};
cudaError_t rtb_launch_query(const QueryParams& Q, int grid, cudaStream_t st);
cudaError_t rtb_launch_unpack(const void* gathered, const UnpackParams& U, cudaStream_t st);
cudaError_t rtb_launch_ffma(float* out, int iters, int grid, cudaStream_t st);
// B0 ceilings (rt_probe.cu)
cudaError_t rtb_probe_ceilings(int num_sms, cudaStream_t st, double out[RT_NUM_CEILINGS]);
cudaError_t rtb_launch_compose(const void* L, const void* R, long long lp, long long rp, int W, int H, int mode,
                               void* out, long long op, cudaStream_t st);
// launchers (rt_build.cu)
size_t rtb_sort_hist_entries(int n);
cudaError_t rtb_build_bvh(const BuildBuffers& B, cudaStream_t st, int* root, int* n_nodes4, int* depth4,
                          int* level_start /* [66] BVH4 node index where each level starts */);
cudaError_t rtb_refit_bvh(float4* prims, float4* nodes4, const int* prim_orig, int n, int n_spheres,
                          const float4* spheres, const uint32_t* tri_idx, const float* vtx,
                          const int* level_start, int levels, cudaStream_t st);
