// rt_api.cu -- host runtime behind the C ABI of include/rt_b200.h.
//
// Owns the per-context CUDA streams (render + copy), the device scene (SoA records + LBVH),
// the camera block, the work counter of the persistent kernel, and the events of the pinned
// download path.  No exception crosses the ABI: every entry point catches and maps to rt_status.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "rt_context.h"

namespace {
thread_local std::string g_err;
}  // namespace

rt_status rtb_fail(rt_status s, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

namespace {

template <typename T>
rt_status dalloc(rt_context* c, size_t count, T** out) {
    *out = nullptr;
    if (count == 0) return RT_OK;
    DevBuf b;
    b.bytes = count * sizeof(T);
    cudaError_t e = cudaMalloc(&b.p, b.bytes);
    if (e != cudaSuccess) return rtb_fail(RT_ERR_OOM, "cudaMalloc(%zu bytes): %s", b.bytes, cudaGetErrorString(e));
    c->scene_bufs.push_back(b);
    *out = static_cast<T*>(b.p);
    return RT_OK;
}

void free_scene(rt_context* c) {
    c->kd_nodes_buf.release();
    c->kd_refs_buf.release();
    for (auto& b : c->scene_bufs) b.release();
    c->scene_bufs.clear();
    c->has_scene = false;
    c->sc = rtb::DevScene{};
}

bool finite3(const float* p) { return std::isfinite(p[0]) && std::isfinite(p[1]) && std::isfinite(p[2]); }

// Block until every render enqueued so far (on any stream) has finished: the scene buffers they
// read may then be freed or rewritten (rt_scene_upload, rt_scene_update_vertices, rt_destroy).
cudaError_t wait_renders(rt_context* c) {
    cudaError_t r = cudaSuccess;
    for (int i = 0; i < RENDER_SLOTS; ++i)
        if (c->slot_used[i]) {
            const cudaError_t e = cudaEventSynchronize(c->slot_ev[i]);
            if (e != cudaSuccess && r == cudaSuccess) r = e;
            c->slot_used[i] = false;
        }
    return r;
}

// Host arrays -> pinned staging -> device, asynchronously on the context stream (SURVEY §8(b):
// "copied to pinned staging").  reserve() sizes the staging once per call; the caller
// synchronises the stream before the staging is reused or the host arrays are released.
struct Stager {
    rt_context* c;
    size_t need = 0, off = 0;
    explicit Stager(rt_context* ctx) : c(ctx) {}
    static size_t pad(size_t b) { return (b + 255) & ~size_t(255); }
    void plan(size_t bytes) { need += pad(bytes); }
    rt_status reserve() {
        if (need <= c->staging_bytes) return RT_OK;
        if (c->staging) cudaFreeHost(c->staging);
        c->staging = nullptr;
        c->staging_bytes = 0;
        const cudaError_t e = cudaHostAlloc(&c->staging, need, cudaHostAllocPortable);
        if (e != cudaSuccess) {
            c->staging = nullptr;
            return rtb_fail(RT_ERR_OOM, "pinned staging cudaHostAlloc(%zu): %s", need, cudaGetErrorString(e));
        }
        c->staging_bytes = need;
        return RT_OK;
    }
    cudaError_t copy(void* dst, const void* src, size_t bytes) {
        if (!bytes) return cudaSuccess;
        char* s = static_cast<char*>(c->staging) + off;
        memcpy(s, src, bytes);
        off += pad(bytes);
        return cudaMemcpyAsync(dst, s, bytes, cudaMemcpyHostToDevice, c->stream);
    }
};

}  // namespace

extern "C" {

int rt_version(void) { return RT_ABI_VERSION; }

int rt_bvh_width(void) { return rtb::BVH_W; }

const char* rt_last_error(void) { return g_err.c_str(); }

rt_status rt_create(int device, void* cuda_stream, rt_context** out) {
    if (!out) return rtb_fail(RT_ERR_INVALID_ARG, "rt_create: out is NULL");
    *out = nullptr;
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return rtb_fail(RT_ERR_INVALID_ARG, "rt_create: device %d of %d", device, ndev);
    rt_context* c = new (std::nothrow) rt_context();
    if (!c) return rtb_fail(RT_ERR_OOM, "rt_create: host allocation");
    c->device = device;
    if (const char* lm = getenv("RT_LEAF_MAX")) c->leaf_max = std::max(1, std::min(16, atoi(lm)));
    if (const char* tp = getenv("RT_TREELETS")) c->treelet_passes = std::max(0, std::min(8, atoi(tp)));
    if (const char* ss = getenv("RT_SAH_SUBTREES")) c->sah_subtrees = std::max(0, std::min(2, atoi(ss)));
    if (const char* sb = getenv("RT_SAH_BIG")) c->sah_big = (int)std::max(2048L, std::min(2147483647L, atol(sb)));
    if (const char* gl = getenv("RT_GRID_LIMIT")) c->grid_limit = std::max(0, atoi(gl));
    if (const char* cd = getenv("RT_COLLAPSE_DP")) c->collapse_dp = atoi(cd) != 0;
    if (const char* cp = getenv("RT_COLLAPSE_CPRIM")) c->collapse_cprim = (float)std::max(0.01, atof(cp));
    if (const char* sm = getenv("RT_SPEC_MASK")) c->spec_mask = atoi(sm) & 7;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess && cuda_stream) {
        c->stream = static_cast<cudaStream_t>(cuda_stream);
    } else if (e == cudaSuccess) {
        e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
        c->own_stream = true;
    }
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->order_ev, cudaEventDisableTiming);
    for (int i = 0; i < RENDER_SLOTS && e == cudaSuccess; ++i)
        e = cudaEventCreateWithFlags(&c->slot_ev[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMalloc(&c->work_counter, 4 * RENDER_SLOTS * sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&c->scratch_counters, RT_NUM_COUNTERS * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMalloc(&c->ffma_out, 64);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) {
        rt_destroy(c);
        return rtb_fail(RT_ERR_CUDA, "rt_create: %s", cudaGetErrorString(e));
    }
    *out = c;
    return RT_OK;
}

rt_status rt_destroy(rt_context* c) {
    if (!c) return RT_OK;
    cudaSetDevice(c->device);
    wait_renders(c);
    rtb_dist_destroy(c);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
    free_scene(c);
    for (auto& e : c->tile_tables) e.buf.release();
    c->tile_tables.clear();
    for (auto& m : c->ipc_maps) cudaIpcCloseMemHandle(m.ptr);
    c->ipc_maps.clear();
    if (c->work_counter) cudaFree(c->work_counter);
    if (c->arena) cudaFree(c->arena);
    if (c->scratch_counters) cudaFree(c->scratch_counters);
    if (c->ffma_out) cudaFree(c->ffma_out);
    if (c->order_ev) cudaEventDestroy(c->order_ev);
    for (auto& ev : c->slot_ev)
        if (ev) cudaEventDestroy(ev);
    if (c->staging) cudaFreeHost(c->staging);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return RT_OK;
}

rt_status rt_synchronize(rt_context* c) {
    if (!c) return rtb_fail(RT_ERR_INVALID_ARG, "rt_synchronize: NULL context");
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->copy_stream));
    return RT_OK;
}

// ------------------------------------------------------------------------------ scene upload
rt_status rt_scene_upload(rt_context* c, const rt_primitives* P, const rt_material* mats, uint32_t n_mats,
                          const rt_light* lights, uint32_t n_lights, const rt_env* env) {
    NvtxRange nvtx_("rt_scene_upload");
    if (!c || !P || !env) return rtb_fail(RT_ERR_INVALID_ARG, "rt_scene_upload: NULL context/primitives/env");
    if ((n_mats && !mats) || (n_lights && !lights))
        return rtb_fail(RT_ERR_INVALID_ARG, "rt_scene_upload: NULL materials/lights with nonzero count");
    const uint32_t S = P->n_spheres, PL = P->n_planes, T = P->n_triangles, V = P->n_vertices;
    if ((S && (!P->spheres || !P->sphere_mat)) || (PL && (!P->planes || !P->plane_mat)) ||
        (T && (!P->tri_indices || !P->tri_mat || !P->vertices)))
        return rtb_fail(RT_ERR_INVALID_ARG, "rt_scene_upload: NULL primitive array with nonzero count");
    if ((uint64_t)S + T >= (1ull << rtb::LEAF_SHIFT) || (uint64_t)S + PL + T >= (1ull << 31))
        return rtb_fail(RT_ERR_INVALID_ARG, "rt_scene_upload: too many primitives (%u spheres + %u triangles)", S, T);
    // ---- validation (SPEC.md:76 ValidationError analogue; SPEC.md:111 degenerate faces)
    for (uint32_t i = 0; i < n_mats; ++i) {
        const rt_material& m = mats[i];
        if (!finite3(m.kd) || !finite3(m.ks) || !std::isfinite(m.shininess) || !std::isfinite(m.kr) ||
            !std::isfinite(m.kt) || !std::isfinite(m.ior))
            return rtb_fail(RT_ERR_INVALID_ARG, "material %u: non-finite value", i);
        for (int k = 0; k < 3; ++k)
            if (m.kd[k] < 0 || m.ks[k] < 0) return rtb_fail(RT_ERR_INVALID_ARG, "material %u: negative kd/ks", i);
        if (m.shininess < 1.0f) return rtb_fail(RT_ERR_INVALID_ARG, "material %u: shininess < 1", i);
        if (m.kr < 0 || m.kr > 1 || m.kt < 0 || m.kt > 1 || m.kr + m.kt > 1.0f)
            return rtb_fail(RT_ERR_INVALID_ARG, "material %u: kr/kt outside [0,1] or kr+kt > 1", i);
        if (!(m.ior > 0)) return rtb_fail(RT_ERR_INVALID_ARG, "material %u: ior <= 0", i);
    }
    for (uint32_t i = 0; i < n_lights; ++i) {
        if (!finite3(lights[i].pos) || !finite3(lights[i].intensity))
            return rtb_fail(RT_ERR_INVALID_ARG, "light %u: non-finite value", i);
        for (int k = 0; k < 3; ++k)
            if (lights[i].intensity[k] < 0) return rtb_fail(RT_ERR_INVALID_ARG, "light %u: negative intensity", i);
    }
    if (!finite3(env->ambient) || !finite3(env->background))
        return rtb_fail(RT_ERR_INVALID_ARG, "env: non-finite ambient/background");
    for (int k = 0; k < 3; ++k)
        if (env->ambient[k] < 0 || env->background[k] < 0)
            return rtb_fail(RT_ERR_INVALID_ARG, "env: negative ambient/background (SPEC.md:35 colours are >= 0)");
    double bound = 0.0;
    for (uint32_t i = 0; i < S; ++i) {
        const float* s = P->spheres + 4 * i;
        if (!finite3(s) || !std::isfinite(s[3])) return rtb_fail(RT_ERR_INVALID_ARG, "sphere %u: non-finite value", i);
        if (!(s[3] > 0)) return rtb_fail(RT_ERR_INVALID_ARG, "sphere %u: radius <= 0", i);
        if (P->sphere_mat[i] >= n_mats) return rtb_fail(RT_ERR_INVALID_ARG, "sphere %u: material %u >= %u", i, P->sphere_mat[i], n_mats);
        bound = std::max(bound, std::fabs((double)s[0]) + std::fabs((double)s[1]) + std::fabs((double)s[2]) + 3.0 * s[3]);
    }
    std::vector<float> planes(4 * (size_t)PL);
    for (uint32_t i = 0; i < PL; ++i) {
        const float* p = P->planes + 4 * i;
        if (!finite3(p) || !std::isfinite(p[3])) return rtb_fail(RT_ERR_INVALID_ARG, "plane %u: non-finite value", i);
        const double n = std::sqrt((double)p[0] * p[0] + (double)p[1] * p[1] + (double)p[2] * p[2]);
        if (!(n > 0)) return rtb_fail(RT_ERR_INVALID_ARG, "plane %u: zero normal", i);
        if (P->plane_mat[i] >= n_mats) return rtb_fail(RT_ERR_INVALID_ARG, "plane %u: material %u >= %u", i, P->plane_mat[i], n_mats);
        for (int k = 0; k < 4; ++k) planes[4 * i + k] = (float)(p[k] / n);
    }
    if (T) {
        for (uint32_t i = 0; i < V; ++i) {
            const float* v = P->vertices + 3 * i;
            if (!finite3(v)) return rtb_fail(RT_ERR_INVALID_ARG, "vertex %u: non-finite value", i);
        }
        for (uint32_t j = 0; j < T; ++j) {
            const uint32_t* t = P->tri_indices + 3 * j;
            if (t[0] >= V || t[1] >= V || t[2] >= V)
                return rtb_fail(RT_ERR_INVALID_ARG, "triangle %u: vertex index >= %u", j, V);
            if (P->tri_mat[j] >= n_mats) return rtb_fail(RT_ERR_INVALID_ARG, "triangle %u: material %u >= %u", j, P->tri_mat[j], n_mats);
            double lo[3], hi[3], e1[3], e2[3];
            for (int k = 0; k < 3; ++k) {
                const double a = P->vertices[3 * t[0] + k], b = P->vertices[3 * t[1] + k], cc = P->vertices[3 * t[2] + k];
                lo[k] = std::min(a, std::min(b, cc));
                hi[k] = std::max(a, std::max(b, cc));
                e1[k] = b - a;
                e2[k] = cc - a;
            }
            const double cx = e1[1] * e2[2] - e1[2] * e2[1], cy = e1[2] * e2[0] - e1[0] * e2[2],
                         cz = e1[0] * e2[1] - e1[1] * e2[0];
            const double area = 0.5 * std::sqrt(cx * cx + cy * cy + cz * cz);
            const double diag2 = (hi[0] - lo[0]) * (hi[0] - lo[0]) + (hi[1] - lo[1]) * (hi[1] - lo[1]) +
                                 (hi[2] - lo[2]) * (hi[2] - lo[2]);
            if (!(area > 1e-12 * diag2)) return rtb_fail(RT_ERR_INVALID_ARG, "triangle %u: degenerate (area %g)", j, area);
        }
        for (uint32_t i = 0; i < V; ++i) {
            const float* v = P->vertices + 3 * i;
            bound = std::max(bound, std::fabs((double)v[0]) + std::fabs((double)v[1]) + std::fabs((double)v[2]));
        }
    }

    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(wait_renders(c));                     // renders in flight on any stream still read the scene
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    free_scene(c);
    const auto t0 = std::chrono::steady_clock::now();
    rt_status st;
    const int N = (int)(S + T);
    // ---- device copies of the raw arrays
    float4* d_spheres = nullptr;
    float* d_vertices = nullptr;
    uint32_t *d_tri = nullptr, *d_trimat = nullptr, *d_smat = nullptr;
    float4* d_planes = nullptr;
    int* d_pmat = nullptr;
    float4 *d_mats = nullptr, *d_lights = nullptr;
    if ((st = dalloc(c, S, &d_spheres)) || (st = dalloc(c, 3 * (size_t)V * (T ? 1 : 0), &d_vertices)) ||
        (st = dalloc(c, 3 * (size_t)T, &d_tri)) || (st = dalloc(c, T, &d_trimat)) || (st = dalloc(c, S, &d_smat)) ||
        (st = dalloc(c, PL, &d_planes)) || (st = dalloc(c, PL, &d_pmat)) || (st = dalloc(c, 3 * (size_t)n_mats, &d_mats)) ||
        (st = dalloc(c, 2 * (size_t)n_lights, &d_lights))) {
        free_scene(c);
        return st;
    }
    // host-side records (planes normalised, materials / lights as float4 rows)
    std::vector<int> pm(PL);
    for (uint32_t i = 0; i < PL; ++i) pm[i] = (int)P->plane_mat[i];
    std::vector<float4> m(3 * (size_t)n_mats);
    for (uint32_t i = 0; i < n_mats; ++i) {
        const rt_material& x = mats[i];
        m[3 * i] = make_float4(x.kd[0], x.kd[1], x.kd[2], x.shininess);
        m[3 * i + 1] = make_float4(x.ks[0], x.ks[1], x.ks[2], x.kr);
        m[3 * i + 2] = make_float4(x.kt, x.ior, 0.f, 0.f);
    }
    std::vector<float4> l(2 * (size_t)n_lights);
    for (uint32_t i = 0; i < n_lights; ++i) {
        l[2 * i] = make_float4(lights[i].pos[0], lights[i].pos[1], lights[i].pos[2], 0.f);
        l[2 * i + 1] = make_float4(lights[i].intensity[0], lights[i].intensity[1], lights[i].intensity[2], 0.f);
    }
    // every array through the pinned staging buffer, DMA'd on the context stream; the build
    // below runs on the same stream, and the stream is synchronised before returning
    {
        Stager sg(c);
        const size_t sz[9] = {16 * (size_t)S, 4 * (size_t)S, T ? 12 * (size_t)V : 0, 12 * (size_t)T, 4 * (size_t)T,
                              16 * (size_t)PL, 4 * (size_t)PL, m.size() * sizeof(float4), l.size() * sizeof(float4)};
        for (size_t b : sz) sg.plan(b);
        if ((st = sg.reserve())) {
            free_scene(c);
            return st;
        }
        CUDA_TRY(sg.copy(d_spheres, P->spheres, sz[0]));
        CUDA_TRY(sg.copy(d_smat, P->sphere_mat, sz[1]));
        CUDA_TRY(sg.copy(d_vertices, P->vertices, sz[2]));
        CUDA_TRY(sg.copy(d_tri, P->tri_indices, sz[3]));
        CUDA_TRY(sg.copy(d_trimat, P->tri_mat, sz[4]));
        CUDA_TRY(sg.copy(d_planes, planes.data(), sz[5]));
        CUDA_TRY(sg.copy(d_pmat, pm.data(), sz[6]));
        CUDA_TRY(sg.copy(d_mats, m.data(), sz[7]));
        CUDA_TRY(sg.copy(d_lights, l.data(), sz[8]));
    }
    // ---- LBVH build buffers
    BuildBuffers B{};
    B.spheres = d_spheres;
    B.vertices = d_vertices;
    B.tri_idx = d_tri;
    B.tri_mat = d_trimat;
    B.sphere_mat = d_smat;
    B.n_spheres = (int)S;
    B.n_planes = (int)PL;
    B.n_tris = (int)T;
    // BVH build scratch: carved from a grow-only per-context arena (no cudaMalloc/cudaFree per
    // upload once it is large enough); sizes are summed in a first pass, pointers set in a second
    size_t arena_off = 0;
    bool measuring = true;
    auto salloc = [&](size_t bytes, void** p) -> rt_status {
        *p = nullptr;
        if (!bytes) return RT_OK;
        const size_t off = arena_off;
        arena_off += (bytes + 255) & ~size_t(255);
        if (!measuring) *p = static_cast<char*>(c->arena) + off;
        return RT_OK;
    };
    float4* d_prims = nullptr;
    float4* d_nodes = nullptr;
    const size_t Nn = N > 1 ? N - 1 : 0;
    int* d_prim_orig = nullptr;
    if ((st = dalloc(c, 3 * (size_t)N, &d_prims)) || (st = dalloc(c, (size_t)N, &d_prim_orig))) {
        free_scene(c);
        return st;
    }
    B.prims = d_prims;
    int root = ~0, n_nodes4 = 0, depth4 = 0;
    B.prim_orig = d_prim_orig;
    std::vector<int> level_start(66, 0);
    if (N > 0) {
        auto alloc_all = [&]() -> rt_status {
            rt_status st2 = RT_OK;
            if ((st2 = salloc(48 * (size_t)N, (void**)&B.prims_unsorted)) || (st2 = salloc(16 * (size_t)N, (void**)&B.aabb_lo)) ||
            (st2 = salloc(16 * (size_t)N, (void**)&B.aabb_hi)) || (st2 = salloc(16 * (size_t)N, (void**)&B.centroid)) ||
            (st2 = salloc(16 * (size_t)N, (void**)&B.leaf_lo)) || (st2 = salloc(16 * (size_t)N, (void**)&B.leaf_hi)) ||
            (st2 = salloc(64, (void**)&B.bounds)) || (st2 = salloc(4 * (size_t)N, (void**)&B.keys[0])) ||
            (st2 = salloc(4 * (size_t)N, (void**)&B.keys[1])) || (st2 = salloc(4 * (size_t)N, (void**)&B.vals[0])) ||
            (st2 = salloc(4 * (size_t)N, (void**)&B.vals[1])) ||
            (st2 = salloc(4 * rtb_sort_hist_entries(N), (void**)&B.hist)) || (st2 = salloc(4 * Nn, (void**)&B.left)) ||
            (st2 = salloc(4 * Nn, (void**)&B.right)) || (st2 = salloc(4 * Nn, (void**)&B.parent_int)) ||
            (st2 = salloc(4 * (size_t)N, (void**)&B.parent_leaf)) || (st2 = salloc(4 * Nn, (void**)&B.flags)) ||
            (st2 = salloc(16 * Nn, (void**)&B.node_lo)) || (st2 = salloc(16 * Nn, (void**)&B.node_hi)) ||
            (st2 = salloc(8 * Nn, (void**)&B.range)) || (st2 = salloc(16 * rtb::NODE_F4 * Nn, (void**)&B.nodes4)) ||
            (st2 = salloc(8 * (size_t)N, (void**)&B.frontier[0])) || (st2 = salloc(8 * (size_t)N, (void**)&B.frontier[1])) ||
            (st2 = salloc(16, (void**)&B.wide_counters)) || (st2 = salloc(4 * Nn, (void**)&B.cost)) ||
            (st2 = salloc(4 * Nn, (void**)&B.count))) {
            return st2;
        }
        return RT_OK;
        };
        alloc_all();                               // measure
        if (arena_off > c->arena_bytes) {
            if (c->arena) cudaFree(c->arena);
            c->arena = nullptr;
            c->arena_bytes = 0;
            cudaError_t ea = cudaMalloc(&c->arena, arena_off);
            if (ea != cudaSuccess) {
                free_scene(c);
                return rtb_fail(RT_ERR_OOM, "BVH scratch arena cudaMalloc(%zu): %s", arena_off, cudaGetErrorString(ea));
            }
            c->arena_bytes = arena_off;
        }
        measuring = false;
        arena_off = 0;
        alloc_all();                               // assign
        B.leaf_max = c->leaf_max;
        B.treelet_passes = c->treelet_passes;
        B.sah_subtrees = c->sah_subtrees;
        B.sah_big = c->sah_big;
        B.collapse_dp = c->collapse_dp;
        B.collapse_cprim = c->collapse_cprim;
        cudaError_t e = rtb_build_bvh(B, c->stream, &root, &n_nodes4, &depth4, level_start.data());
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
        if (e == cudaSuccess && n_nodes4 > 0) {        // compact the BVH4 into an exact-size buffer
            if ((st = dalloc(c, rtb::NODE_F4 * (size_t)n_nodes4, &d_nodes))) {
                free_scene(c);
                return st;
            }
            e = cudaMemcpyAsync(d_nodes, B.nodes4, 16 * rtb::NODE_F4 * (size_t)n_nodes4, cudaMemcpyDeviceToDevice,
                                c->stream);
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);   // staging and build scratch free again
        if (e != cudaSuccess) {
            free_scene(c);
            return rtb_fail(RT_ERR_CUDA, "LBVH build: %s", cudaGetErrorString(e));
        }
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));       // the staged copies have landed (N == 0 case)
    const auto t1 = std::chrono::steady_clock::now();

    rtb::DevScene& D = c->sc;
    D.nodes = d_nodes;
    D.prims = d_prims;
    D.planes = d_planes;
    D.plane_mat = d_pmat;
    D.mats = d_mats;
    D.lights = d_lights;
    D.n_bvh = N;
    D.root = root;
    D.n_spheres = (int)S;
    D.n_planes = (int)PL;
    D.n_lights = (int)n_lights;
    D.refractive = 0;
    for (uint32_t i = 0; i < n_mats; ++i) D.refractive |= mats[i].kt > 0.0f;
    D.bound = (float)(bound * (1.0 + 1e-6));
    D.ambient = make_float3(env->ambient[0], env->ambient[1], env->ambient[2]);
    D.background = make_float3(env->background[0], env->background[1], env->background[2]);
    size_t bytes = 0;
    for (auto& b : c->scene_bufs) bytes += b.bytes;
    c->info[0] = S;
    c->info[1] = PL;
    c->info[2] = T;
    c->info[3] = N;
    c->info[4] = (uint64_t)n_nodes4;
    c->info[5] = (uint64_t)depth4;
    c->info[6] = bytes;
    c->info[7] = (uint64_t)std::chrono::duration_cast<std::chrono::microseconds>(t1 - t0).count();
    // kept for rt_scene_update_vertices (NEXT-3 refit)
    c->d_prim_orig = d_prim_orig;
    c->scene_leaf_max = c->leaf_max;                 // the leaf bound this scene's BVH was built with
    c->d_vertices = d_vertices;
    c->d_tri = d_tri;
    c->d_spheres = d_spheres;
    c->n_vertices = T ? V : 0;
    c->level_start.assign(level_start.begin(), level_start.begin() + std::min(66, depth4 + 1));
    c->sphere_bound = 0.0;
    for (uint32_t i = 0; i < S; ++i) {
        const float* sp = P->spheres + 4 * i;
        c->sphere_bound = std::max(c->sphere_bound, std::fabs((double)sp[0]) + std::fabs((double)sp[1]) +
                                                        std::fabs((double)sp[2]) + 3.0 * sp[3]);
    }
    if (T) c->h_tri.assign(P->tri_indices, P->tri_indices + 3 * (size_t)T);
    else c->h_tri.clear();
    c->has_scene = true;
    return RT_OK;
}

// ------------------------------------------------------------------------------ refit (NEXT-3)
rt_status rt_scene_update_vertices(rt_context* c, const float* vertices, uint32_t n_vertices) {
    NvtxRange nvtx_("rt_scene_update_vertices");
    if (!c || (!vertices && n_vertices)) return rtb_fail(RT_ERR_INVALID_ARG, "rt_scene_update_vertices: NULL argument");
    if (!c->has_scene) return rtb_fail(RT_ERR_NO_SCENE, "rt_scene_update_vertices: no scene");
    if (n_vertices != c->n_vertices)
        return rtb_fail(RT_ERR_INVALID_ARG, "rt_scene_update_vertices: %u vertices, scene has %u", n_vertices, c->n_vertices);
    if (n_vertices == 0) return RT_OK;
    double bound = c->sphere_bound;
    for (uint32_t i = 0; i < n_vertices; ++i) {
        const float* v = vertices + 3 * i;
        if (!finite3(v)) return rtb_fail(RT_ERR_INVALID_ARG, "vertex %u: non-finite value", i);
        bound = std::max(bound, std::fabs((double)v[0]) + std::fabs((double)v[1]) + std::fabs((double)v[2]));
    }
    const size_t T = c->h_tri.size() / 3;
    for (size_t j = 0; j < T; ++j) {                    // SPEC.md:111 degenerate faces stay rejected
        const uint32_t* t = c->h_tri.data() + 3 * j;
        double lo[3], hi[3], e1[3], e2[3];
        for (int k = 0; k < 3; ++k) {
            const double a = vertices[3 * t[0] + k], b = vertices[3 * t[1] + k], cc = vertices[3 * t[2] + k];
            lo[k] = std::min(a, std::min(b, cc));
            hi[k] = std::max(a, std::max(b, cc));
            e1[k] = b - a;
            e2[k] = cc - a;
        }
        const double cx = e1[1] * e2[2] - e1[2] * e2[1], cy = e1[2] * e2[0] - e1[0] * e2[2], cz = e1[0] * e2[1] - e1[1] * e2[0];
        const double area = 0.5 * std::sqrt(cx * cx + cy * cy + cz * cz);
        const double diag2 = (hi[0] - lo[0]) * (hi[0] - lo[0]) + (hi[1] - lo[1]) * (hi[1] - lo[1]) + (hi[2] - lo[2]) * (hi[2] - lo[2]);
        if (!(area > 1e-12 * diag2)) return rtb_fail(RT_ERR_INVALID_ARG, "triangle %zu: degenerate after update", j);
    }
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(wait_renders(c));                     // renders in flight read the nodes the refit rewrites
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    {
        Stager sg(c);
        sg.plan(12 * (size_t)n_vertices);
        rt_status st;
        if ((st = sg.reserve())) return st;
        CUDA_TRY(sg.copy(c->d_vertices, vertices, 12 * (size_t)n_vertices));
    }
    CUDA_TRY(rtb_refit_bvh(const_cast<float4*>(c->sc.prims), const_cast<float4*>(c->sc.nodes), c->d_prim_orig,
                           c->sc.n_bvh, c->sc.n_spheres, c->d_spheres, c->d_tri, c->d_vertices, c->level_start.data(),
                           (int)c->level_start.size() - 1, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));       // host vertices may be freed on return
    c->sc.bound = (float)(bound * (1.0 + 1e-6));
    return RT_OK;
}

// ------------------------------------------------------------------------------ camera
rt_status rt_set_stereo_camera(rt_context* c, const float eye[3], const float look_at[3], const float up[3],
                               float vfov_deg, float interocular, float convergence) {
    if (!c || !eye || !look_at || !up) return rtb_fail(RT_ERR_INVALID_ARG, "rt_set_stereo_camera: NULL argument");
    if (!finite3(eye) || !finite3(look_at) || !finite3(up) || !std::isfinite(vfov_deg) || !std::isfinite(interocular) ||
        std::isnan(convergence) || convergence == -INFINITY)
        return rtb_fail(RT_ERR_INVALID_ARG, "rt_set_stereo_camera: non-finite input");
    if (!(vfov_deg > 0.0f && vfov_deg < 180.0f)) return rtb_fail(RT_ERR_INVALID_ARG, "vfov %g outside (0,180)", vfov_deg);
    if (interocular < 0.0f) return rtb_fail(RT_ERR_INVALID_ARG, "negative interocular distance");
    // SPEC.md:425 (derive_eyes), in double
    double f[3] = {(double)look_at[0] - eye[0], (double)look_at[1] - eye[1], (double)look_at[2] - eye[2]};
    const double fl = std::sqrt(f[0] * f[0] + f[1] * f[1] + f[2] * f[2]);
    if (!(fl > 0)) return rtb_fail(RT_ERR_INVALID_ARG, "eye == look_at");
    for (double& x : f) x /= fl;
    double r[3] = {f[1] * up[2] - f[2] * up[1], f[2] * up[0] - f[0] * up[2], f[0] * up[1] - f[1] * up[0]};
    const double rl = std::sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    if (!(rl > 0)) return rtb_fail(RT_ERR_INVALID_ARG, "up is parallel to the view direction");
    for (double& x : r) x /= rl;
    const double u[3] = {r[1] * f[2] - r[2] * f[1], r[2] * f[0] - r[0] * f[2], r[0] * f[1] - r[1] * f[0]};
    const double s = interocular;
    for (int k = 0; k < 3; ++k) {
        c->cam_eye[0][k] = eye[k] - 0.5 * s * r[k];
        c->cam_eye[1][k] = eye[k] + 0.5 * s * r[k];
        c->cam_f[k] = f[k];
        c->cam_r[k] = r[k];
        c->cam_u[k] = u[k];
    }
    c->cam_th = std::tan(0.5 * (double)vfov_deg * M_PI / 180.0);
    c->cam_sigma_unit = (convergence > 0.0f && std::isfinite(convergence)) ? s / (2.0 * convergence) : 0.0;
    c->has_camera = true;
    return RT_OK;
}

}  // extern "C"

namespace {

rt_status fill_camera(rt_context* c, uint32_t W, uint32_t H, rtb::DevCamera& cam) {
    for (int e = 0; e < 2; ++e)
        cam.eye[e] = make_float3((float)c->cam_eye[e][0], (float)c->cam_eye[e][1], (float)c->cam_eye[e][2]);
    cam.f = make_float3((float)c->cam_f[0], (float)c->cam_f[1], (float)c->cam_f[2]);
    cam.r = make_float3((float)c->cam_r[0], (float)c->cam_r[1], (float)c->cam_r[2]);
    cam.u = make_float3((float)c->cam_u[0], (float)c->cam_u[1], (float)c->cam_u[2]);
    cam.th = (float)c->cam_th;
    cam.tha = (float)(c->cam_th * (double)W / (double)H);
    cam.sigma[0] = (float)(+c->cam_sigma_unit);
    cam.sigma[1] = (float)(-c->cam_sigma_unit);
    return RT_OK;
}

struct ShardGeom {
    int tiles_x, tiles_y, tiles_per_eye, mode;
    int block;              // mode 2: tile pairs dealt in B x B blocks of tiles (1 = single tiles)
};

ShardGeom shard_geom(uint32_t W, uint32_t H, uint32_t world) {
    ShardGeom g;
    g.tiles_x = (int)((W + RT_TILE - 1) / RT_TILE);
    g.tiles_y = (int)((H + RT_TILE - 1) / RT_TILE);
    g.tiles_per_eye = g.tiles_x * g.tiles_y;
    // 1: eye split; 0 / 2: tile pairs round-robin.  RT_SHARD_PAIRS=1 (experiment knob; every
    // rank and the root must see the same value) deals tile pairs at world 2 as well.
    static const bool pairs_at_2 = [] { const char* e = getenv("RT_SHARD_PAIRS"); return e && atoi(e) != 0; }();
    g.mode = world == 1 ? 0 : (world == 2 && !pairs_at_2 ? 1 : 2);
    // RT_SHARD_BLOCK=B (read once per process; every rank must see the same value): tile pairs are
    // dealt to ranks in B x B blocks of tiles (raster order of blocks, block b -> rank b mod world),
    // so a rank's tiles are spatially compact; 1 (default) = single tiles round-robin
    static const int block = [] { const char* e = getenv("RT_SHARD_BLOCK"); return e ? std::max(1, atoi(e)) : 1; }();
    g.block = g.mode == 2 ? block : 1;
    return g;
}

// mode 2 with blocks: this rank's tile indices (raster order inside each of its blocks)
std::vector<uint32_t> block_tiles(const ShardGeom& g, uint32_t rank, uint32_t world) {
    std::vector<uint32_t> t;
    const int B = g.block, nbx = (g.tiles_x + B - 1) / B, nby = (g.tiles_y + B - 1) / B;
    for (int b = (int)rank; b < nbx * nby; b += (int)world) {
        const int bx = b % nbx, by = b / nbx;
        for (int y = by * B; y < std::min(g.tiles_y, by * B + B); ++y)
            for (int x = bx * B; x < std::min(g.tiles_x, bx * B + B); ++x) t.push_back((uint32_t)(y * g.tiles_x + x));
    }
    return t;
}

uint32_t shard_count(const ShardGeom& g, uint32_t rank, uint32_t world) {
    if (g.mode == 1) return (uint32_t)g.tiles_per_eye;
    if (g.block > 1) return 2u * (uint32_t)block_tiles(g, rank, world).size();
    const int pairs = (int)rank < g.tiles_per_eye ? (g.tiles_per_eye - (int)rank + (int)world - 1) / (int)world : 0;
    return 2u * (uint32_t)pairs;
}

// global tile id G: eye = G & 1, tile = G >> 1 (eyes interleaved)
uint32_t shard_tile(const ShardGeom& g, uint32_t rank, uint32_t world, uint32_t lt) {
    if (g.mode == 1) return 2u * lt + rank;
    if (g.block > 1) return 2u * block_tiles(g, rank, world)[lt >> 1] + (lt & 1u);
    return 2u * (rank + (lt >> 1) * world) + (lt & 1u);
}

// device copy of a tile table (cached per layout): one rank's tiles (render) or every rank's,
// padded with -1 to the largest rank (unpack)
rt_status tile_table(rt_context* c, const ShardGeom& g, uint32_t W, uint32_t H, int rank, uint32_t world, uint32_t pad,
                     const int** out) {
    for (auto& e : c->tile_tables)
        if (e.W == W && e.H == H && e.rank == rank && e.world == world && e.block == g.block) {
            *out = static_cast<const int*>(e.buf.p);
            return RT_OK;
        }
    std::vector<int> h;
    for (uint32_t r = (rank < 0 ? 0u : (uint32_t)rank); r < (rank < 0 ? world : (uint32_t)rank + 1); ++r) {
        const std::vector<uint32_t> t = block_tiles(g, r, world);
        for (uint32_t x : t) h.push_back((int)x);
        for (size_t k = t.size(); rank < 0 && k < pad; ++k) h.push_back(-1);
    }
    if (h.empty()) h.push_back(-1);
    RtTileTable e;
    e.W = W; e.H = H; e.rank = rank; e.world = world; e.block = g.block;
    e.buf.bytes = h.size() * sizeof(int);
    CUDA_TRY(cudaMalloc(&e.buf.p, e.buf.bytes));
    // once per layout; a pageable cudaMemcpy may return before its DMA lands and is not ordered
    // with the (non-blocking) render streams, so copy on the context stream and wait for it
    cudaError_t ce = cudaMemcpyAsync(e.buf.p, h.data(), e.buf.bytes, cudaMemcpyHostToDevice, c->stream);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(c->stream);
    if (ce != cudaSuccess) {
        cudaFree(e.buf.p);
        return rtb_fail(RT_ERR_CUDA, "tile table upload: %s", cudaGetErrorString(ce));
    }
    c->tile_tables.push_back(e);
    *out = static_cast<const int*>(e.buf.p);
    return RT_OK;
}

rt_status check_fb(const rt_fb& fb, uint32_t W, const char* name) {
    if (!fb.dev_ptr) return RT_OK;
    if (fb.format != RT_FORMAT_RGBA8 && fb.format != RT_FORMAT_RGBA16F)
        return rtb_fail(RT_ERR_INVALID_ARG, "%s: unknown format %u", name, fb.format);
    const uint64_t need = (uint64_t)W * (fb.format == RT_FORMAT_RGBA8 ? 4 : 8);
    if (fb.pitch_bytes < need) return rtb_fail(RT_ERR_SIZE, "%s: pitch %llu < %llu", name, (unsigned long long)fb.pitch_bytes, (unsigned long long)need);
    if (fb.pitch_bytes % (fb.format == RT_FORMAT_RGBA8 ? 4 : 8))
        return rtb_fail(RT_ERR_INVALID_ARG, "%s: pitch not a multiple of the pixel size", name);
    return RT_OK;
}

}  // namespace

extern "C" {

rt_status rt_render_stereo_ex(rt_context* c, const rt_render_params* p, const rt_outputs* out) {
    NvtxRange nvtx_("rt_render_stereo_ex");
    if (!c || !p || !out) return rtb_fail(RT_ERR_INVALID_ARG, "rt_render_stereo_ex: NULL argument");
    if (c->dist) return rtb_dist_render(c, p, out, c->stream);
    return rtb_render_local(c, p, out, c->stream);
}

rt_status rt_render_stereo_async(rt_context* c, const rt_render_params* p, const rt_outputs* out, void* cuda_stream) {
    NvtxRange nvtx_("rt_render_stereo_async");
    if (!c || !p || !out) return rtb_fail(RT_ERR_INVALID_ARG, "rt_render_stereo_async: NULL argument");
    cudaStream_t st = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : c->stream;
    if (c->dist) return rtb_dist_render(c, p, out, st);
    return rtb_render_local(c, p, out, st);
}

}  // extern "C"

rt_status rtb_render_local(rt_context* c, const rt_render_params* p, const rt_outputs* out, cudaStream_t stream) {
    if (!c->has_scene) return rtb_fail(RT_ERR_NO_SCENE, "render before rt_scene_upload");
    if (!c->has_camera) return rtb_fail(RT_ERR_NO_CAMERA, "render before rt_set_stereo_camera");
    const uint32_t W = p->width, H = p->height;
    if (W == 0 || H == 0 || W > 16384 || H > 16384) return rtb_fail(RT_ERR_SIZE, "image size %ux%u", W, H);
    if (p->max_depth > RT_MAX_DEPTH) return rtb_fail(RT_ERR_SIZE, "max_depth %u > %d", p->max_depth, RT_MAX_DEPTH);
    if (p->shard_world == 0 || p->shard_rank >= p->shard_world || p->shard_world > 4096)
        return rtb_fail(RT_ERR_INVALID_ARG, "shard %u of %u", p->shard_rank, p->shard_world);
    if (p->flags & ~(RT_RENDER_COUNT | RT_RENDER_BRUTE_FORCE | RT_RENDER_PEER_STORE | RT_RENDER_KDTREE))
        return rtb_fail(RT_ERR_INVALID_ARG, "unknown flags 0x%x", p->flags);
    if ((p->flags & RT_RENDER_KDTREE) && (p->flags & RT_RENDER_BRUTE_FORCE))
        return rtb_fail(RT_ERR_INVALID_ARG, "RT_RENDER_KDTREE and RT_RENDER_BRUTE_FORCE are exclusive");
    if ((p->flags & RT_RENDER_KDTREE) && c->sc.n_bvh > 0 && !c->sc.kd_nodes)
        return rtb_fail(RT_ERR_INVALID_ARG, "RT_RENDER_KDTREE needs rt_kdtree_build after the upload");
    if ((p->flags & RT_RENDER_COUNT) && !out->counters) return rtb_fail(RT_ERR_INVALID_ARG, "RT_RENDER_COUNT needs counters");
    rt_status st;
    if ((st = check_fb(out->left, W, "out_left")) || (st = check_fb(out->right, W, "out_right"))) return st;
    if (out->shard && out->shard_format != RT_FORMAT_RGBA8 && out->shard_format != RT_FORMAT_RGBA16F)
        return rtb_fail(RT_ERR_INVALID_ARG, "shard: unknown format");
    TraceParams P{};
    P.sc = c->sc;
    fill_camera(c, W, H, P.cam);
    P.W = (int)W;
    P.H = (int)H;
    P.max_depth = (int)p->max_depth;
    // a work counter per render in flight (RENDER_SLOTS slots, rotated): renders enqueued on
    // different streams may run concurrently and must not share a queue; a render that reuses a
    // slot waits on the device for the slot's previous render (launch below)
    const int slot = (int)(c->render_seq % RENDER_SLOTS);
    P.work_counter = c->work_counter + 4 * slot;
    const ShardGeom g = shard_geom(W, H, p->shard_world);
    const uint64_t n_tiles = shard_count(g, p->shard_rank, p->shard_world);
    if (n_tiles * 256ull >= (1ull << 31)) return rtb_fail(RT_ERR_SIZE, "too many pixels in one shard");
    P.n_work = (int)(n_tiles * 256);
    P.tiles_x = g.tiles_x;
    P.tiles_per_eye = g.tiles_per_eye;
    P.shard_mode = g.mode;
    P.shard_rank = (int)p->shard_rank;
    P.shard_world = (int)p->shard_world;
    P.tile_list = nullptr;
    if (g.mode == 2 && g.block > 1) {
        CUDA_TRY(cudaSetDevice(c->device));
        if ((st = tile_table(c, g, W, H, (int)p->shard_rank, p->shard_world, 0, &P.tile_list))) return st;
    }
    P.fb[0] = out->left.dev_ptr;
    P.fb[1] = out->right.dev_ptr;
    P.fb_fmt[0] = (int)out->left.format;
    P.fb_fmt[1] = (int)out->right.format;
    P.fb_pitch[0] = (long long)out->left.pitch_bytes;
    P.fb_pitch[1] = (long long)out->right.pitch_bytes;
    P.prim_id = out->prim_id;
    P.radiance = reinterpret_cast<float4*>(out->radiance);
    P.shard = out->shard;
    P.shard_fmt = (int)out->shard_format;
    P.counters = out->counters ? out->counters : c->scratch_counters;
    P.stack_entries = (rtb::BVH_W - 1) * (int)c->info[5] + 2;   // <= W-1 pending siblings per level
    if (P.stack_entries > rtb::STACK_CAP) return rtb_fail(RT_ERR_SIZE, "BVH too deep (%d levels)", (int)c->info[5]);
    P.n_tiles = (int)n_tiles;
    P.peer_fence = (p->flags & RT_RENDER_PEER_STORE) ? 1 : 0;
    for (int e = 0; e < 2; ++e)
        P.fb_vec[e] = P.fb[e] && ((uintptr_t)P.fb[e] % 16 == 0) && (P.fb_pitch[e] % 16 == 0);
    if (out->composed.dev_ptr) {
        if (out->composed.format != RT_FORMAT_RGBA8) return rtb_fail(RT_ERR_INVALID_ARG, "composed: RGBA8 only");
        if (out->compose_mode != RT_COMPOSE_ANAGLYPH && out->compose_mode != RT_COMPOSE_SBS)
            return rtb_fail(RT_ERR_INVALID_ARG, "composed: mode %u", out->compose_mode);
        if (g.mode == 1) return rtb_fail(RT_ERR_INVALID_ARG, "composed: the world-2 eye split traces one eye per launch");
        if (p->flags & (RT_RENDER_COUNT | RT_RENDER_BRUTE_FORCE | RT_RENDER_KDTREE))
            return rtb_fail(RT_ERR_INVALID_ARG, "composed: product renders only (no COUNT / BRUTE_FORCE / KDTREE)");
        if (out->compose_mode == RT_COMPOSE_SBS && W < 2) return rtb_fail(RT_ERR_INVALID_ARG, "composed: SBS needs width >= 2");
        const uint32_t cw = out->compose_mode == RT_COMPOSE_ANAGLYPH ? W : 2 * (W / 2);
        if ((st = check_fb(out->composed, cw, "composed"))) return st;
        P.comp = out->composed.dev_ptr;
        P.comp_pitch = (long long)out->composed.pitch_bytes;
        P.comp_mode = (int)out->compose_mode;
        P.comp_vec = ((uintptr_t)P.comp % 16 == 0) && (P.comp_pitch % 16 == 0);
    }
    if (P.n_work == 0) return RT_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    int occ = 0;
    unsigned kflags = P.comp ? RTB_TRACE_COMPOSE : (p->flags & (RT_RENDER_COUNT | RT_RENDER_BRUTE_FORCE | RT_RENDER_KDTREE));
    if (!(kflags & (RT_RENDER_COUNT | RT_RENDER_BRUTE_FORCE | RT_RENDER_KDTREE))) {
        // product launches: the instantiation without the code this scene can never take
        if ((c->spec_mask & 1) && P.sc.n_spheres == 0 && P.sc.n_planes == 0) kflags |= RTB_TRACE_TRI;
        if ((c->spec_mask & 2) && !P.sc.refractive) kflags |= RTB_TRACE_OPAQUE;
        if ((c->spec_mask & 4) && c->scene_leaf_max == 1) kflags |= RTB_TRACE_LEAF1;
    }
    CUDA_TRY(rtb_trace_occupancy(kflags, P.stack_entries, &occ));
    if (occ < 1) occ = 1;
    const int block = rtb_trace_block();
    const long long max_blocks = ((long long)P.n_work + block - 1) / block;
    int grid = (int)std::min<long long>((long long)c->num_sms * occ, std::max<long long>(1, max_blocks));
    if (c->grid_limit > 0) grid = std::min(grid, c->grid_limit);   // experiment knob (paper's "network size")
    if (c->slot_used[slot]) CUDA_TRY(cudaStreamWaitEvent(stream, c->slot_ev[slot], 0));
    CUDA_TRY(cudaMemsetAsync(P.work_counter, 0, sizeof(int), stream));
    CUDA_TRY(rtb_launch_trace(P, kflags, grid, stream));
    CUDA_TRY(cudaEventRecord(c->slot_ev[slot], stream));
    c->slot_used[slot] = true;
    ++c->render_seq;
    return RT_OK;
}
extern "C" {

rt_status rt_render_stereo(rt_context* c, uint32_t width, uint32_t height, uint32_t max_depth, rt_fb out_left,
                           rt_fb out_right) {
    rt_render_params p{};
    p.width = width;
    p.height = height;
    p.max_depth = max_depth;
    p.shard_rank = 0;
    p.shard_world = 1;
    rt_outputs o{};
    o.left = out_left;
    o.right = out_right;
    return rt_render_stereo_ex(c, &p, &o);
}

// ------------------------------------------------------------------------------ download
rt_status rt_host_alloc(size_t bytes, void** out) {
    if (!out || !bytes) return rtb_fail(RT_ERR_INVALID_ARG, "rt_host_alloc: NULL out or zero size");
    cudaError_t e = cudaHostAlloc(out, bytes, cudaHostAllocPortable);
    if (e != cudaSuccess) {
        *out = nullptr;
        return rtb_fail(RT_ERR_OOM, "cudaHostAlloc(%zu): %s", bytes, cudaGetErrorString(e));
    }
    return RT_OK;
}

rt_status rt_host_free(void* p) {
    if (!p) return RT_OK;
    CUDA_TRY(cudaFreeHost(p));
    return RT_OK;
}

static bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

rt_status rt_download(rt_context* c, const void* dev_src, void* host_dst, size_t bytes, rt_event** done) {
    return rt_download_after(c, dev_src, host_dst, bytes, nullptr, done);
}

rt_status rt_download_after(rt_context* c, const void* dev_src, void* host_dst, size_t bytes, void* after_stream,
                            rt_event** done) {
    NvtxRange nvtx_("rt_download");
    if (done) *done = nullptr;
    if (!c || !dev_src || !host_dst || !bytes) return rtb_fail(RT_ERR_INVALID_ARG, "rt_download: NULL pointer or zero size");
    CUDA_TRY(cudaSetDevice(c->device));
    if (!is_pinned(host_dst)) return rtb_fail(RT_ERR_INVALID_ARG, "rt_download: host_dst is not pinned host memory");
    CUDA_TRY(cudaEventRecord(c->order_ev, after_stream ? static_cast<cudaStream_t>(after_stream) : c->stream));
    CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->order_ev, 0));
    CUDA_TRY(cudaMemcpyAsync(host_dst, dev_src, bytes, cudaMemcpyDeviceToHost, c->copy_stream));
    if (done) {
        rt_event* ev = new (std::nothrow) rt_event();
        if (!ev) return rtb_fail(RT_ERR_OOM, "rt_download: event allocation");
        cudaError_t e = cudaEventCreateWithFlags(&ev->ev, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventRecord(ev->ev, c->copy_stream);
        if (e != cudaSuccess) {
            if (ev->ev) cudaEventDestroy(ev->ev);
            delete ev;
            return rtb_fail(RT_ERR_CUDA, "rt_download: %s", cudaGetErrorString(e));
        }
        *done = ev;
    }
    return RT_OK;
}

rt_status rt_upload(rt_context* c, const void* host_src, void* dev_dst, size_t bytes) {
    if (!c || !host_src || !dev_dst || !bytes) return rtb_fail(RT_ERR_INVALID_ARG, "rt_upload: NULL pointer or zero size");
    CUDA_TRY(cudaSetDevice(c->device));
    if (!is_pinned(host_src)) return rtb_fail(RT_ERR_INVALID_ARG, "rt_upload: host_src is not pinned host memory");
    CUDA_TRY(cudaMemcpyAsync(dev_dst, host_src, bytes, cudaMemcpyHostToDevice, c->stream));
    return RT_OK;
}

rt_status rt_wait(rt_event* ev) {
    if (!ev) return rtb_fail(RT_ERR_INVALID_ARG, "rt_wait: NULL event");
    cudaError_t e = cudaEventSynchronize(ev->ev);
    cudaEventDestroy(ev->ev);
    delete ev;
    if (e != cudaSuccess) return rtb_fail(RT_ERR_CUDA, "rt_wait: %s", cudaGetErrorString(e));
    return RT_OK;
}

rt_status rt_query(rt_event* ev) {
    if (!ev) return rtb_fail(RT_ERR_INVALID_ARG, "rt_query: NULL event");
    cudaError_t e = cudaEventQuery(ev->ev);
    if (e == cudaSuccess) return RT_OK;
    if (e == cudaErrorNotReady) {
        cudaGetLastError();
        return RT_ERR_NOT_READY;
    }
    return rtb_fail(RT_ERR_CUDA, "rt_query: %s", cudaGetErrorString(e));
}

// ------------------------------------------------------------------------------ shards
rt_status rt_shard_tiles(uint32_t W, uint32_t H, uint32_t rank, uint32_t world, uint32_t* n_tiles, uint32_t* ids) {
    if (!n_tiles || W == 0 || H == 0 || world == 0 || rank >= world || W > 16384 || H > 16384)
        return rtb_fail(RT_ERR_INVALID_ARG, "rt_shard_tiles: bad arguments");
    const ShardGeom g = shard_geom(W, H, world);
    const uint32_t n = shard_count(g, rank, world);
    if (ids)
        for (uint32_t lt = 0; lt < n; ++lt) ids[lt] = shard_tile(g, rank, world, lt);
    *n_tiles = n;
    return RT_OK;
}

rt_status rt_shard_bytes(uint32_t W, uint32_t H, uint32_t world, uint32_t format, uint64_t* bytes) {
    if (!bytes || W == 0 || H == 0 || world == 0 || (format != RT_FORMAT_RGBA8 && format != RT_FORMAT_RGBA16F))
        return rtb_fail(RT_ERR_INVALID_ARG, "rt_shard_bytes: bad arguments");
    const ShardGeom g = shard_geom(W, H, world);
    uint32_t mx = 0;
    for (uint32_t r = 0; r < world; ++r) mx = std::max(mx, shard_count(g, r, world));
    *bytes = (uint64_t)mx * 256u * (format == RT_FORMAT_RGBA8 ? 4u : 8u);
    return RT_OK;
}

rt_status rt_unpack_shards_host(const void* gathered, uint32_t W, uint32_t H, uint32_t world, uint32_t format,
                                void* left, void* right, uint64_t pitch) {
    uint64_t per = 0;
    rt_status st = rt_shard_bytes(W, H, world, format, &per);
    if (st) return st;
    if (!gathered) return rtb_fail(RT_ERR_INVALID_ARG, "rt_unpack_shards_host: NULL gathered");
    const uint32_t bpp = format == RT_FORMAT_RGBA8 ? 4 : 8;
    if (pitch < (uint64_t)W * bpp) return rtb_fail(RT_ERR_SIZE, "rt_unpack_shards_host: pitch too small");
    const ShardGeom g = shard_geom(W, H, world);
    const char* src = static_cast<const char*>(gathered);
    for (uint32_t r = 0; r < world; ++r) {
        const uint32_t n = shard_count(g, r, world);
        for (uint32_t lt = 0; lt < n; ++lt) {
            const uint32_t gt = shard_tile(g, r, world, lt);
            const int eye = (int)(gt & 1u);
            const int t = (int)(gt >> 1);
            char* dst = static_cast<char*>(eye ? right : left);
            if (!dst) continue;
            for (int w = 0; w < 256; ++w) {
                const int px = (t % g.tiles_x) * RT_TILE + w % RT_TILE;
                const int py = (t / g.tiles_x) * RT_TILE + w / RT_TILE;
                if (px >= (int)W || py >= (int)H) continue;
                memcpy(dst + (uint64_t)py * pitch + (uint64_t)px * bpp,
                       src + r * per + ((uint64_t)lt * 256 + w) * bpp, bpp);
            }
        }
    }
    return RT_OK;
}

rt_status rt_unpack_shards(rt_context* c, const void* gathered, uint32_t W, uint32_t H, uint32_t world, uint32_t format,
                           rt_fb left, rt_fb right) {
    NvtxRange nvtx_("rt_unpack_shards");
    if (!c || !gathered) return rtb_fail(RT_ERR_INVALID_ARG, "rt_unpack_shards: NULL argument");
    return rtb_unpack_on(c, gathered, W, H, world, format, left, right, c->stream);
}

}  // extern "C"

rt_status rtb_unpack_on(rt_context* c, const void* gathered, uint32_t W, uint32_t H, uint32_t world, uint32_t format,
                        rt_fb left, rt_fb right, cudaStream_t stream) {
    uint64_t per = 0;
    rt_status st = rt_shard_bytes(W, H, world, format, &per);
    if (st) return st;
    if ((left.dev_ptr && left.format != format) || (right.dev_ptr && right.format != format))
        return rtb_fail(RT_ERR_INVALID_ARG, "rt_unpack_shards: framebuffer format differs from the shard format");
    if (left.dev_ptr && right.dev_ptr && left.pitch_bytes != right.pitch_bytes)
        return rtb_fail(RT_ERR_INVALID_ARG, "rt_unpack_shards: left/right pitch differ");
    if ((st = check_fb(left, W, "left")) || (st = check_fb(right, W, "right"))) return st;
    const ShardGeom g = shard_geom(W, H, world);
    UnpackParams U{};
    U.left = left.dev_ptr;
    U.right = right.dev_ptr;
    U.pitch = (long long)(left.dev_ptr ? left.pitch_bytes : right.pitch_bytes);
    U.fmt = (int)format;
    U.W = (int)W;
    U.H = (int)H;
    U.tiles_x = g.tiles_x;
    U.tiles_per_eye = g.tiles_per_eye;
    U.tiles_per_rank = (int)(per / (256u * (format == RT_FORMAT_RGBA8 ? 4u : 8u)));
    U.world = (int)world;
    U.shard_mode = g.mode;
    U.gtile = nullptr;
    CUDA_TRY(cudaSetDevice(c->device));
    if (g.mode == 2 && g.block > 1 && (st = tile_table(c, g, W, H, -1, world, (uint32_t)U.tiles_per_rank / 2, &U.gtile)))
        return st;
    CUDA_TRY(rtb_launch_unpack(gathered, U, stream));
    return RT_OK;
}

extern "C" {

// ------------------------------------------------------------------------------ peer memory
rt_status rt_ipc_get_handle(const void* dev_ptr, void* handle64, uint64_t* offset) {
    if (!dev_ptr || !handle64 || !offset) return rtb_fail(RT_ERR_INVALID_ARG, "rt_ipc_get_handle: NULL argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    // driver entry point through the runtime (the library does not link libcuda directly)
    using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
        return rtb_fail(RT_ERR_PEER, "cuMemGetAddressRange entry point unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    CUresult r = reinterpret_cast<GetRange>(fn)(&base, &size, (CUdeviceptr)dev_ptr);
    if (r != CUDA_SUCCESS) return rtb_fail(RT_ERR_PEER, "cuMemGetAddressRange failed (%d)", (int)r);
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) return rtb_fail(RT_ERR_PEER, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    memcpy(handle64, &h, 64);
    *offset = (uint64_t)((CUdeviceptr)dev_ptr - base);
    return RT_OK;
}

rt_status rt_ipc_open(rt_context* c, const void* handle64, void** dev_ptr) {
    if (!c || !handle64 || !dev_ptr) return rtb_fail(RT_ERR_INVALID_ARG, "rt_ipc_open: NULL argument");
    CUDA_TRY(cudaSetDevice(c->device));
    // one mapping per exported allocation per process: several framebuffers can share one
    // caching-allocator block (one handle, different offsets), and CUDA maps a handle once
    std::string key(static_cast<const char*>(handle64), 64);
    for (auto& m : c->ipc_maps)
        if (m.key == key) {
            ++m.refs;
            *dev_ptr = m.ptr;
            return RT_OK;
        }
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return rtb_fail(RT_ERR_PEER, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    c->ipc_maps.push_back({key, *dev_ptr, 1});
    return RT_OK;
}

rt_status rt_ipc_close(rt_context* c, void* dev_ptr) {
    if (!c || !dev_ptr) return rtb_fail(RT_ERR_INVALID_ARG, "rt_ipc_close: NULL argument");
    CUDA_TRY(cudaSetDevice(c->device));
    for (size_t i = 0; i < c->ipc_maps.size(); ++i)
        if (c->ipc_maps[i].ptr == dev_ptr) {
            if (--c->ipc_maps[i].refs > 0) return RT_OK;
            c->ipc_maps.erase(c->ipc_maps.begin() + (long)i);
            break;
        }
    cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    if (e != cudaSuccess) return rtb_fail(RT_ERR_PEER, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
    return RT_OK;
}

// ------------------------------------------------------------------------------ composition
rt_status rt_compose(rt_context* c, rt_fb left, rt_fb right, uint32_t W, uint32_t H, uint32_t mode, rt_fb out) {
    NvtxRange nvtx_("rt_compose");
    if (!c || !left.dev_ptr || !right.dev_ptr || !out.dev_ptr) return rtb_fail(RT_ERR_INVALID_ARG, "rt_compose: NULL argument");
    if (left.format != RT_FORMAT_RGBA8 || right.format != RT_FORMAT_RGBA8 || out.format != RT_FORMAT_RGBA8)
        return rtb_fail(RT_ERR_INVALID_ARG, "rt_compose: RGBA8 framebuffers only");
    if (mode != RT_COMPOSE_ANAGLYPH && mode != RT_COMPOSE_SBS) return rtb_fail(RT_ERR_INVALID_ARG, "rt_compose: mode %u", mode);
    if (W == 0 || H == 0 || W > 16384 || H > 16384) return rtb_fail(RT_ERR_SIZE, "rt_compose: size %ux%u", W, H);
    if (mode == RT_COMPOSE_SBS && W < 2) return rtb_fail(RT_ERR_INVALID_ARG, "rt_compose: SBS needs width >= 2");
    const uint64_t out_w = mode == RT_COMPOSE_ANAGLYPH ? W : 2 * (W / 2);
    rt_status st;
    if ((st = check_fb(left, W, "left")) || (st = check_fb(right, W, "right")) || (st = check_fb(out, (uint32_t)out_w, "out")))
        return st;
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(rtb_launch_compose(left.dev_ptr, right.dev_ptr, (long long)left.pitch_bytes, (long long)right.pitch_bytes,
                                (int)W, (int)H, (int)mode, out.dev_ptr, (long long)out.pitch_bytes, c->stream));
    return RT_OK;
}

// ------------------------------------------------------------------------------ introspection
rt_status rt_kdtree_build(rt_context* c, uint32_t max_leaf, uint32_t max_depth, uint64_t info[6]) {
    NvtxRange nvtx_("rt_kdtree_build");
    if (!c) return rtb_fail(RT_ERR_INVALID_ARG, "rt_kdtree_build: NULL context");
    if (max_leaf < 1 || max_leaf > 4096) return rtb_fail(RT_ERR_INVALID_ARG, "rt_kdtree_build: max_leaf %u", max_leaf);
    if (max_depth > 60) return rtb_fail(RT_ERR_INVALID_ARG, "rt_kdtree_build: max_depth %u > 60", max_depth);
    if (!c->has_scene) return rtb_fail(RT_ERR_NO_SCENE, "rt_kdtree_build: no scene");
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(wait_renders(c));                     // kd renders in flight read the buffers replaced below
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    const int n = c->sc.n_bvh;
    const auto t0 = std::chrono::steady_clock::now();
    rtb::KdHost K;
    if (n > 0) {
        std::vector<float4> prims(3 * (size_t)n);
        CUDA_TRY(cudaMemcpyAsync(prims.data(), c->sc.prims, prims.size() * sizeof(float4), cudaMemcpyDeviceToHost,
                                 c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        rtb::kd_build_host(prims.data(), n, c->sc.n_spheres, (int)max_leaf, (int)max_depth, K);
    }
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    c->kd_nodes_buf.release();
    c->kd_refs_buf.release();
    c->sc.kd_nodes = nullptr;
    c->sc.kd_refs = nullptr;
    if (n > 0) {
        DevBuf a, b;
        a.bytes = K.nodes.size() * sizeof(int2);
        b.bytes = std::max<size_t>(K.refs.size(), 1) * sizeof(int);
        cudaError_t e = cudaMalloc(&a.p, a.bytes);
        if (e == cudaSuccess) e = cudaMalloc(&b.p, b.bytes);
        if (e != cudaSuccess) {
            a.release();
            b.release();
            return rtb_fail(RT_ERR_OOM, "rt_kdtree_build: cudaMalloc: %s", cudaGetErrorString(e));
        }
        c->kd_nodes_buf = a;
        c->kd_refs_buf = b;
        CUDA_TRY(cudaMemcpyAsync(a.p, K.nodes.data(), a.bytes, cudaMemcpyHostToDevice, c->stream));
        if (!K.refs.empty())
            CUDA_TRY(cudaMemcpyAsync(b.p, K.refs.data(), K.refs.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));       // pageable sources: complete before they go away
        c->sc.kd_nodes = static_cast<const int2*>(a.p);
        c->sc.kd_refs = static_cast<const int*>(b.p);
        c->sc.kd_lo = make_float3(K.lo[0], K.lo[1], K.lo[2]);
        c->sc.kd_hi = make_float3(K.hi[0], K.hi[1], K.hi[2]);
    }
    if (info) {
        info[0] = K.nodes.size();
        info[1] = K.refs.size();
        info[2] = (uint64_t)K.depth;
        info[3] = (uint64_t)K.leaves;
        info[4] = K.nodes.size() * sizeof(int2) + K.refs.size() * sizeof(int);
        info[5] = (uint64_t)us;
    }
    return RT_OK;
}

rt_status rt_scene_info(rt_context* c, uint64_t info[8]) {
    if (!c || !info) return rtb_fail(RT_ERR_INVALID_ARG, "rt_scene_info: NULL argument");
    if (!c->has_scene) return rtb_fail(RT_ERR_NO_SCENE, "rt_scene_info: no scene");
    memcpy(info, c->info, sizeof c->info);
    return RT_OK;
}

rt_status rt_intersect(rt_context* c, const float* o, const float* d, const float* tmax, uint32_t n, uint32_t flags,
                       float* out_t, int32_t* out_id, void* stream) {
    if (!c) return rtb_fail(RT_ERR_INVALID_ARG, "rt_intersect: NULL context");
    if (flags & ~(RT_QUERY_ANY | RT_QUERY_BRUTE_FORCE)) return rtb_fail(RT_ERR_INVALID_ARG, "rt_intersect: flags 0x%x", flags);
    const bool any = flags & RT_QUERY_ANY;
    if (n && (!o || !d || !out_id || (any && !tmax) || (!any && !out_t)))
        return rtb_fail(RT_ERR_INVALID_ARG, "rt_intersect: NULL array");
    if (!c->has_scene) return rtb_fail(RT_ERR_NO_SCENE, "rt_intersect: no scene");
    if (n == 0) return RT_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    QueryParams Q;
    Q.sc = c->sc;
    Q.o = o;
    Q.d = d;
    Q.tmax = tmax;
    Q.out_t = out_t;
    Q.out_id = out_id;
    Q.n = n;
    Q.any = any;
    Q.brute = (flags & RT_QUERY_BRUTE_FORCE) != 0;
    const int block = rtb_trace_block();
    const int grid = (int)std::min<long long>((long long)c->num_sms * 16, ((long long)n + block - 1) / block);
    CUDA_TRY(rtb_launch_query(Q, grid, stream ? static_cast<cudaStream_t>(stream) : c->stream));
    return RT_OK;
}

rt_status rt_bvh_export(rt_context* c, float* nodes, uint32_t* n_nodes, int32_t* prim_gid, uint32_t* n_prims) {
    if (!c || !n_nodes || !n_prims) return rtb_fail(RT_ERR_INVALID_ARG, "rt_bvh_export: NULL argument");
    if (!c->has_scene) return rtb_fail(RT_ERR_NO_SCENE, "rt_bvh_export: no scene");
    const uint32_t nn = (uint32_t)c->info[4], np = (uint32_t)c->sc.n_bvh;
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (nodes && nn) {
        CUDA_TRY(cudaMemcpy2D(nodes, 16 * rtb::NODE_DATA_F4, c->sc.nodes, 16 * rtb::NODE_F4, 16 * rtb::NODE_DATA_F4, nn,
                              cudaMemcpyDeviceToHost));
        if (rtb::node_slot(6) != 6) {       // device slot order -> the documented export order
            // (plain float copies: the caller's array need not be 16-byte aligned)
            constexpr int A = rtb::BVH_W;                     // floats per array (lo.x[W] ...)
            float tmp[7 * A];
            for (uint32_t i = 0; i < nn; ++i) {
                float* q = nodes + (size_t)i * 7 * A;
                for (int a = 0; a < 7; ++a) memcpy(tmp + a * A, q + rtb::node_slot(a) * A, sizeof(float) * A);
                memcpy(q, tmp, sizeof tmp);
            }
        }
    }
    if (prim_gid && np) {
        std::vector<float4> p(3 * (size_t)np);
        CUDA_TRY(cudaMemcpy(p.data(), c->sc.prims, p.size() * sizeof(float4), cudaMemcpyDeviceToHost));
        for (uint32_t k = 0; k < np; ++k) {
            int32_t g;
            memcpy(&g, &p[3 * k].w, 4);
            prim_gid[k] = g;
        }
    }
    *n_nodes = nn;
    *n_prims = np;
    return RT_OK;
}

rt_status rt_bench_ffma(rt_context* c, uint32_t iters, double* tflops, double* ms) {
    if (!c || !tflops || !ms || !iters) return rtb_fail(RT_ERR_INVALID_ARG, "rt_bench_ffma: bad argument");
    CUDA_TRY(cudaSetDevice(c->device));
    const int grid = c->num_sms * 8;
    cudaEvent_t a, b;
    CUDA_TRY(cudaEventCreate(&a));
    CUDA_TRY(cudaEventCreate(&b));
    CUDA_TRY(rtb_launch_ffma(c->ffma_out, (int)iters, grid, c->stream));   // warm-up
    CUDA_TRY(cudaEventRecord(a, c->stream));
    CUDA_TRY(rtb_launch_ffma(c->ffma_out, (int)iters, grid, c->stream));
    CUDA_TRY(cudaEventRecord(b, c->stream));
    CUDA_TRY(cudaEventSynchronize(b));
    float t = 0;
    CUDA_TRY(cudaEventElapsedTime(&t, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    const double flops = 2.0 * 8 * 16 * (double)iters * grid * 256;
    *ms = t;
    *tflops = flops / (t * 1e-3) / 1e12;
    return RT_OK;
}

rt_status rt_bench_ceilings(rt_context* c, double out[RT_NUM_CEILINGS]) {
    if (!c || !out) return rtb_fail(RT_ERR_INVALID_ARG, "rt_bench_ceilings: NULL argument");
    CUDA_TRY(cudaSetDevice(c->device));
    for (int i = 0; i < RT_NUM_CEILINGS; ++i) out[i] = 0.0;
    CUDA_TRY(rtb_probe_ceilings(c->num_sms, c->stream, out));
    return RT_OK;
}

}  // extern "C"
