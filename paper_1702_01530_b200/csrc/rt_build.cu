// rt_build.cu -- device-side scene packing and Morton-code LBVH construction.
//
// SURVEY.md §8(a) rows a1-a2; PAPER.md:44 (Table 1: BVH "high speed and adaptability of
// construction", "good for the GPU").  Steps, all on the device:
//   k_prim_setup     triangles -> (v0, e1, e2) records, spheres -> (c, r, r^2) records, AABBs, centroids
//   k_bounds         centroid bounds (order-independent min/max -> deterministic)
//   k_morton         30-bit Morton code (10 bits per axis) of the normalised centroid
//   radix sort       hand-written stable LSD sort, 4 passes of 8/8/8/6 bits, ties keep the
//                    original primitive order -> the 64-bit key (morton << 32 | position) is unique
//   k_karras         Karras 2012 hierarchy: each internal node finds its key range and split
//                    from common-prefix lengths (__clzll)
//   k_refit          bottom-up AABB union with atomic arrival counters
//   k_gather_prims   primitive records in leaf order
//   k_sah_level      maximal subtrees of <= 16384 primitives rebuilt by binned SAH, all at once,
//                    level by level, one warp per node (k_sah_roots finds them, k_sah_init seeds)
//   k_treelets       SAH treelet restructuring of the BVH2 (Karras & Aila 2013), optional passes
//   k_wide           BVH2 -> 4-wide BVH collapse (level by level), small subtrees -> leaves
// The result is a deterministic function of the input arrays.
#include <cfloat>

#include "rt_device.cuh"
#include <cstdlib>
#include <vector>

#include "rt_internal.h"

namespace rtb {

constexpr int SORT_THREADS = 256;
constexpr int SORT_ITEMS = 8;
constexpr int SORT_TILE = SORT_THREADS * SORT_ITEMS;

__device__ __forceinline__ unsigned int f2ord(float f) {
    const unsigned int u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned int u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

__global__ void k_prim_setup(BuildBuffers B) {
    const int N = B.n_spheres + B.n_tris;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        float4 r0, r1, r2, lo, hi, ce;
        if (i < B.n_spheres) {
            const float4 s = B.spheres[i];
            r0 = make_float4(s.x, s.y, s.z, __int_as_float(i));
            r1 = make_float4(s.w, s.w * s.w, 0.0f, __int_as_float((int)B.sphere_mat[i]));
            r2 = make_float4(s.w * s.w, 0.f, 0.f, 0.f);          // r^2 again: the test reads records 0 and 2
            // round outward so the box contains the sphere
            lo = make_float4(__fsub_rd(s.x, s.w), __fsub_rd(s.y, s.w), __fsub_rd(s.z, s.w), 0.f);
            hi = make_float4(__fadd_ru(s.x, s.w), __fadd_ru(s.y, s.w), __fadd_ru(s.z, s.w), 0.f);
            ce = make_float4(s.x, s.y, s.z, 0.f);
        } else {
            const int j = i - B.n_spheres;
            const uint32_t a = B.tri_idx[3 * j], b = B.tri_idx[3 * j + 1], c = B.tri_idx[3 * j + 2];
            const float3 v0 = f3(B.vertices[3 * a], B.vertices[3 * a + 1], B.vertices[3 * a + 2]);
            const float3 v1 = f3(B.vertices[3 * b], B.vertices[3 * b + 1], B.vertices[3 * b + 2]);
            const float3 v2 = f3(B.vertices[3 * c], B.vertices[3 * c + 1], B.vertices[3 * c + 2]);
            const int gid = B.n_spheres + B.n_planes + j;
            r0 = make_float4(v0.x, v0.y, v0.z, __int_as_float(gid));
            r1 = make_float4(v1.x - v0.x, v1.y - v0.y, v1.z - v0.z, __int_as_float((int)B.tri_mat[j]));
            r2 = make_float4(v2.x - v0.x, v2.y - v0.y, v2.z - v0.z, 0.f);
            lo = make_float4(fminf(v0.x, fminf(v1.x, v2.x)), fminf(v0.y, fminf(v1.y, v2.y)),
                             fminf(v0.z, fminf(v1.z, v2.z)), 0.f);
            hi = make_float4(fmaxf(v0.x, fmaxf(v1.x, v2.x)), fmaxf(v0.y, fmaxf(v1.y, v2.y)),
                             fmaxf(v0.z, fmaxf(v1.z, v2.z)), 0.f);
            ce = make_float4((v0.x + v1.x + v2.x) * (1.0f / 3.0f), (v0.y + v1.y + v2.y) * (1.0f / 3.0f),
                             (v0.z + v1.z + v2.z) * (1.0f / 3.0f), 0.f);
        }
        B.prims_unsorted[3 * i] = r0;
        B.prims_unsorted[3 * i + 1] = r1;
        B.prims_unsorted[3 * i + 2] = r2;
        B.aabb_lo[i] = lo;
        B.aabb_hi[i] = hi;
        B.centroid[i] = ce;
    }
}

__global__ void k_bounds_init(unsigned int* b) {
    if (threadIdx.x < 3) b[threadIdx.x] = f2ord(FLT_MAX);
    else if (threadIdx.x < 6) b[threadIdx.x] = f2ord(-FLT_MAX);
}

__global__ void k_bounds(const float4* __restrict__ ce, int n, unsigned int* b) {
    float mn[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, mx[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float4 c = ce[i];
        mn[0] = fminf(mn[0], c.x); mn[1] = fminf(mn[1], c.y); mn[2] = fminf(mn[2], c.z);
        mx[0] = fmaxf(mx[0], c.x); mx[1] = fmaxf(mx[1], c.y); mx[2] = fmaxf(mx[2], c.z);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            mn[k] = fminf(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], off));
            mx[k] = fmaxf(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], off));
        }
    }
    if ((threadIdx.x & 31) == 0) {
        for (int k = 0; k < 3; ++k) {
            atomicMin(&b[k], f2ord(mn[k]));
            atomicMax(&b[3 + k], f2ord(mx[k]));
        }
    }
}

__device__ __forceinline__ uint32_t expand_bits10(uint32_t v) {
    v = (v * 0x00010001u) & 0xFF0000FFu;
    v = (v * 0x00000101u) & 0x0F00F00Fu;
    v = (v * 0x00000011u) & 0xC30C30C3u;
    v = (v * 0x00000005u) & 0x49249249u;
    return v;
}

__global__ void k_morton(const float4* __restrict__ ce, int n, const unsigned int* b, uint32_t* keys, uint32_t* vals) {
    const float lo[3] = {ord2f(b[0]), ord2f(b[1]), ord2f(b[2])};
    const float hi[3] = {ord2f(b[3]), ord2f(b[4]), ord2f(b[5])};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float4 c = ce[i];
        const float v[3] = {c.x, c.y, c.z};
        uint32_t q[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float ext = hi[k] - lo[k];
            const float u = ext > 0.0f ? (v[k] - lo[k]) / ext : 0.5f;
            q[k] = (uint32_t)fminf(fmaxf(u * 1024.0f, 0.0f), 1023.0f);
        }
        keys[i] = (expand_bits10(q[0]) << 2) | (expand_bits10(q[1]) << 1) | expand_bits10(q[2]);
        vals[i] = (uint32_t)i;
    }
}

// ---------------------------------------------------------------- stable LSD radix sort
__global__ void __launch_bounds__(SORT_THREADS) k_radix_hist(const uint32_t* __restrict__ keys, int n, int shift,
                                                           uint32_t* hist, int nblocks) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int base = blockIdx.x * SORT_TILE;
#pragma unroll
    for (int i = 0; i < SORT_ITEMS; ++i) {
        const int idx = base + i * SORT_THREADS + threadIdx.x;
        if (idx < n) atomicAdd(&h[(keys[idx] >> shift) & 255u], 1u);
    }
    __syncthreads();
    hist[threadIdx.x * nblocks + blockIdx.x] = h[threadIdx.x];
}

// Exclusive scan of `n` entries with one block of 1024 threads (n is ~256 * N/2048), 8 consecutive
// entries per thread a step (round 1: one entry per thread, 113 us for C4's 125 K entries).
__global__ void __launch_bounds__(1024) k_scan_single(uint32_t* a, int n) {
    constexpr int IPT = 8;                               // the vector path below assumes 8
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int base = 0; base < n; base += 1024 * IPT) {
        const int i0 = base + threadIdx.x * IPT;
        uint32_t v[IPT], t = 0;
        if (i0 + IPT <= n && (reinterpret_cast<uintptr_t>(a) & 15u) == 0) {   // two 16-byte loads
            const uint4 x0 = reinterpret_cast<const uint4*>(a + i0)[0], x1 = reinterpret_cast<const uint4*>(a + i0)[1];
            v[0] = x0.x; v[1] = x0.y; v[2] = x0.z; v[3] = x0.w; v[4] = x1.x; v[5] = x1.y; v[6] = x1.z; v[7] = x1.w;
        } else {
#pragma unroll
            for (int k = 0; k < IPT; ++k) v[k] = i0 + k < n ? a[i0 + k] : 0u;
        }
#pragma unroll
        for (int k = 0; k < IPT; ++k) t += v[k];
        uint32_t x = t;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
            if (lane >= off) x += y;
        }
        if (lane == 31) warp_sums[wid] = x;
        __syncthreads();
        if (wid == 0) {
            uint32_t s = warp_sums[lane];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, s, off);
                if (lane >= off) s += y;
            }
            warp_sums[lane] = s;
        }
        __syncthreads();
        uint32_t run = x - t + (wid ? warp_sums[wid - 1] : 0u) + carry;
        uint32_t o[IPT];
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            o[k] = run;
            run += v[k];
        }
        if (i0 + IPT <= n && (reinterpret_cast<uintptr_t>(a) & 15u) == 0) {
            reinterpret_cast<uint4*>(a + i0)[0] = make_uint4(o[0], o[1], o[2], o[3]);
            reinterpret_cast<uint4*>(a + i0)[1] = make_uint4(o[4], o[5], o[6], o[7]);
        } else {
#pragma unroll
            for (int k = 0; k < IPT; ++k)
                if (i0 + k < n) a[i0 + k] = o[k];
        }
        __syncthreads();
        if (threadIdx.x == 1023) carry = run;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(SORT_THREADS) k_radix_scatter(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                              uint32_t* kout, uint32_t* vout, int n, int shift,
                                                              const uint32_t* __restrict__ hist, int nblocks) {
    constexpr int NW = SORT_THREADS / 32;
    __shared__ uint32_t goff[256];
    __shared__ uint32_t wcnt[NW][256];
    __shared__ uint32_t woff[NW][256];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    goff[threadIdx.x] = hist[threadIdx.x * nblocks + blockIdx.x];
    const int base = blockIdx.x * SORT_TILE;
    const uint32_t lt_mask = (1u << lane) - 1u;
    for (int it = 0; it < SORT_ITEMS; ++it) {
#pragma unroll
        for (int w = 0; w < NW; ++w) wcnt[w][threadIdx.x] = 0;
        __syncthreads();
        const int idx = base + it * SORT_THREADS + threadIdx.x;
        const bool valid = idx < n;
        uint32_t key = 0, val = 0, dig = 0xFFFFFFFFu;
        if (valid) { key = kin[idx]; val = vin[idx]; dig = (key >> shift) & 255u; }
        const uint32_t peers = __match_any_sync(0xffffffffu, dig);
        const uint32_t rank = __popc(peers & lt_mask);
        if (valid && rank == 0) wcnt[wid][dig] = __popc(peers);
        __syncthreads();
        {
            const int d = threadIdx.x;
            uint32_t run = goff[d];
#pragma unroll
            for (int w = 0; w < NW; ++w) { woff[w][d] = run; run += wcnt[w][d]; }
            goff[d] = run;
        }
        __syncthreads();
        if (valid) {
            const uint32_t pos = woff[wid][dig] + rank;
            kout[pos] = key;
            vout[pos] = val;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- Karras hierarchy
__device__ __forceinline__ int delta(const uint32_t* __restrict__ keys, int n, int i, int j) {
    if (j < 0 || j >= n) return -1;
    const unsigned long long a = ((unsigned long long)keys[i] << 32) | (unsigned)i;
    const unsigned long long b = ((unsigned long long)keys[j] << 32) | (unsigned)j;
    return __clzll(a ^ b);
}

__global__ void k_karras(const uint32_t* __restrict__ keys, int n, int* left, int* right, int* parent_int, int* parent_leaf,
                         int2* range) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n - 1; i += gridDim.x * blockDim.x) {
        const int d = (delta(keys, n, i, i + 1) - delta(keys, n, i, i - 1)) >= 0 ? 1 : -1;
        const int dmin = delta(keys, n, i, i - d);
        int lmax = 2;
        while (delta(keys, n, i, i + lmax * d) > dmin) lmax <<= 1;
        int l = 0;
        for (int t = lmax >> 1; t >= 1; t >>= 1)
            if (delta(keys, n, i, i + (l + t) * d) > dmin) l += t;
        const int j = i + l * d;
        const int first = min(i, j), last = max(i, j);
        const int dnode = delta(keys, n, first, last);
        int split = first, step = last - first;
        do {
            step = (step + 1) >> 1;
            const int ns = split + step;
            if (ns < last && delta(keys, n, first, ns) > dnode) split = ns;
        } while (step > 1);
        int lc, rc;
        if (split == first) { lc = ~split; parent_leaf[split] = i; }          // leaf: ~slot (count 1)
        else { lc = split; parent_int[split] = i; }
        if (split + 1 == last) { rc = ~(split + 1); parent_leaf[split + 1] = i; }
        else { rc = split + 1; parent_int[split + 1] = i; }
        left[i] = lc;
        right[i] = rc;
        range[i] = make_int2(first, last);
        if (i == 0) parent_int[0] = -1;
    }
}

__device__ __forceinline__ void child_box(int c, const float4* lo_leaf, const float4* hi_leaf, const float4* lo_int,
                                          const float4* hi_int, float4& lo, float4& hi) {
    if (c < 0) { lo = lo_leaf[~c]; hi = hi_leaf[~c]; }
    else { lo = __ldcg(&lo_int[c]); hi = __ldcg(&hi_int[c]); }
}

__global__ void k_refit(BuildBuffers B, int n, const float4* __restrict__ slo, const float4* __restrict__ shi) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        int p = B.parent_leaf[k];
        while (p >= 0) {
            __threadfence();
            if (atomicAdd(&B.flags[p], 1) == 0) break;    // first arrival: the sibling finishes p
            __threadfence();
            float4 a0, a1, b0, b1;
            child_box(B.left[p], slo, shi, B.node_lo, B.node_hi, a0, a1);
            child_box(B.right[p], slo, shi, B.node_lo, B.node_hi, b0, b1);
            __stcg(&B.node_lo[p], make_float4(fminf(a0.x, b0.x), fminf(a0.y, b0.y), fminf(a0.z, b0.z), 0.f));
            __stcg(&B.node_hi[p], make_float4(fmaxf(a1.x, b1.x), fmaxf(a1.y, b1.y), fmaxf(a1.z, b1.z), 0.f));
            p = B.parent_int[p];
        }
    }
}

// ---------------------------------------------------------------- treelet restructuring
// Karras & Aila 2013 (TRBVH), one thread per treelet: bottom-up (atomic arrival counters as
// in k_refit); at every internal node with >= 7 primitives the treelet of 7 leaves is formed by
// repeatedly opening the largest-area treelet leaf, the SAH-optimal binary topology over the 7
// leaves is found by dynamic programming over all 127 subsets, and the treelet's 6 internal
// nodes are rewired when that lowers the SAH cost.  Leaf order (Morton) and the root index are
// unchanged; only parent/child links, boxes, costs and counts of treelet nodes change.
constexpr float SAH_CI = 1.2f;   // internal-node (box test) cost
constexpr float SAH_CT = 1.0f;   // primitive test cost

__device__ __forceinline__ float area3(float3 lo, float3 hi) {
    const float x = hi.x - lo.x, y = hi.y - lo.y, z = hi.z - lo.z;
    return x * y + y * z + z * x;
}

struct TNode {
    float3 lo, hi;
    float cost;
    int count;
};

__device__ __forceinline__ TNode tnode(const BuildBuffers& B, int code) {
    TNode t;
    if (code < 0) {
        const float4 a = B.leaf_lo[~code], b = B.leaf_hi[~code];
        t.lo = f3(a.x, a.y, a.z);
        t.hi = f3(b.x, b.y, b.z);
        t.cost = SAH_CT * area3(t.lo, t.hi);
        t.count = 1;
    } else {
        const float4 a = __ldcg(&B.node_lo[code]), b = __ldcg(&B.node_hi[code]);
        t.lo = f3(a.x, a.y, a.z);
        t.hi = f3(b.x, b.y, b.z);
        t.cost = __ldcg(&B.cost[code]);
        t.count = __ldcg(&B.count[code]);
    }
    return t;
}

__device__ __forceinline__ void set_parent(const BuildBuffers& B, int child, int parent) {
    if (child < 0) __stcg(&B.parent_leaf[~child], parent);
    else __stcg(&B.parent_int[child], parent);
}

__device__ void treelet_node(const BuildBuffers& B, int p) {
    const int l = __ldcg(&B.left[p]), r = __ldcg(&B.right[p]);
    const TNode tl = tnode(B, l), tr = tnode(B, r);
    const int cnt = tl.count + tr.count;
    const float3 plo = f3(fminf(tl.lo.x, tr.lo.x), fminf(tl.lo.y, tr.lo.y), fminf(tl.lo.z, tr.lo.z));
    const float3 phi = f3(fmaxf(tl.hi.x, tr.hi.x), fmaxf(tl.hi.y, tr.hi.y), fmaxf(tl.hi.z, tr.hi.z));
    const float pcost = SAH_CI * area3(plo, phi) + tl.cost + tr.cost;
    bool done = false;
    if (cnt >= 7) {
        int leaves[7], inner[6];
        TNode lt[7];
        int nl = 2, ni = 1;
        inner[0] = p;
        leaves[0] = l; lt[0] = tl;
        leaves[1] = r; lt[1] = tr;
        while (nl < 7) {
            int best = -1;
            float ba = -1.0f;
            for (int i = 0; i < nl; ++i)
                if (leaves[i] >= 0) {
                    const float a = area3(lt[i].lo, lt[i].hi);
                    if (a > ba) { ba = a; best = i; }
                }
            if (best < 0) break;
            const int c = leaves[best];
            inner[ni++] = c;
            const int cl = __ldcg(&B.left[c]), cr = __ldcg(&B.right[c]);
            leaves[best] = cl; lt[best] = tnode(B, cl);
            leaves[nl] = cr; lt[nl] = tnode(B, cr);
            ++nl;
        }
        if (nl == 7) {
            float sa[128], copt[128];
            unsigned char part[128];
            for (int s = 1; s < 128; ++s) {
                float3 lo = f3(3.4e38f, 3.4e38f, 3.4e38f), hi = f3(-3.4e38f, -3.4e38f, -3.4e38f);
                for (int i = 0; i < 7; ++i)
                    if (s & (1 << i)) {
                        lo = f3(fminf(lo.x, lt[i].lo.x), fminf(lo.y, lt[i].lo.y), fminf(lo.z, lt[i].lo.z));
                        hi = f3(fmaxf(hi.x, lt[i].hi.x), fmaxf(hi.y, lt[i].hi.y), fmaxf(hi.z, lt[i].hi.z));
                    }
                sa[s] = area3(lo, hi);
            }
            for (int s = 1; s < 128; ++s) {
                if (__popc(s) == 1) {
                    copt[s] = lt[__ffs(s) - 1].cost;
                    part[s] = 0;
                    continue;
                }
                const int low = s & -s, rest = s ^ low;
                float best = 3.4e38f;
                int bt = low;
                for (int tp = rest;; tp = (tp - 1) & rest) {
                    const int t = tp | low;
                    if (t != s) {
                        const float c = copt[t] + copt[s ^ t];
                        if (c < best) { best = c; bt = t; }
                    }
                    if (tp == 0) break;
                }
                copt[s] = SAH_CI * sa[s] + best;
                part[s] = (unsigned char)bt;
            }
            if (copt[127] < pcost * (1.0f - 1e-5f)) {
                // rewire: depth-first over the optimal partition, reusing the 6 inner nodes
                int st_s[7], st_n[7], sp = 0, next = 1;
                st_s[sp] = 127; st_n[sp] = p; ++sp;
                while (sp > 0) {
                    --sp;
                    const int sset = st_s[sp], node = st_n[sp];
                    const int halves[2] = {part[sset], sset ^ part[sset]};
                    int codes[2];
                    for (int h = 0; h < 2; ++h) {
                        if (__popc(halves[h]) == 1) {
                            codes[h] = leaves[__ffs(halves[h]) - 1];
                        } else {
                            codes[h] = inner[next++];
                            st_s[sp] = halves[h]; st_n[sp] = codes[h]; ++sp;
                        }
                        set_parent(B, codes[h], node);
                    }
                    __stcg(&B.left[node], codes[0]);
                    __stcg(&B.right[node], codes[1]);
                    float3 lo = f3(3.4e38f, 3.4e38f, 3.4e38f), hi = f3(-3.4e38f, -3.4e38f, -3.4e38f);
                    int c = 0;
                    for (int i = 0; i < 7; ++i)
                        if (sset & (1 << i)) {
                            lo = f3(fminf(lo.x, lt[i].lo.x), fminf(lo.y, lt[i].lo.y), fminf(lo.z, lt[i].lo.z));
                            hi = f3(fmaxf(hi.x, lt[i].hi.x), fmaxf(hi.y, lt[i].hi.y), fmaxf(hi.z, lt[i].hi.z));
                            c += lt[i].count;
                        }
                    __stcg(&B.node_lo[node], make_float4(lo.x, lo.y, lo.z, 0.f));
                    __stcg(&B.node_hi[node], make_float4(hi.x, hi.y, hi.z, 0.f));
                    __stcg(&B.cost[node], copt[sset]);
                    __stcg(&B.count[node], c);
                }
                done = true;
            }
        }
    }
    if (!done) {
        __stcg(&B.node_lo[p], make_float4(plo.x, plo.y, plo.z, 0.f));
        __stcg(&B.node_hi[p], make_float4(phi.x, phi.y, phi.z, 0.f));
        __stcg(&B.cost[p], pcost);
        __stcg(&B.count[p], cnt);
    }
}

__global__ void k_treelets(BuildBuffers B, int n) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        int p = __ldcg(&B.parent_leaf[k]);
        while (p >= 0) {
            __threadfence();
            if (atomicAdd(&B.flags[p], 1) == 0) break;    // first arrival: the sibling finishes p
            __threadfence();
            treelet_node(B, p);
            __threadfence();
            p = __ldcg(&B.parent_int[p]);
        }
    }
}

// ---------------------------------------------------------------- BVH2 -> BVH4 collapse
// Node layout (rt_device.cuh): 7 float4 = lo.x[4] hi.x[4] lo.y[4] hi.y[4] lo.z[4] hi.z[4] child[4].
// A BVH2 internal child covering <= leaf_max primitives becomes a leaf over its contiguous
// (Morton-sorted) range.  Each BVH4 node starts from the two children of one BVH2 node and
// greedily opens the internal child with the largest surface area until it has 4 children.
struct WChild {
    int code;      // BVH2: >= 0 internal node, < 0 ~leaf-slot; after finalize: BVH4 code
    float4 lo, hi;
};

__device__ __forceinline__ float half_area(float4 lo, float4 hi) {
    const float x = hi.x - lo.x, y = hi.y - lo.y, z = hi.z - lo.z;
    return x * y + y * z + z * x;
}

__device__ __forceinline__ bool is_open(int code, const int2* __restrict__ range, int leaf_max) {
    if (code < 0) return false;
    const int2 r = range[code];
    return r.y - r.x + 1 > leaf_max;
}

__device__ __forceinline__ WChild make_child(int code, const BuildBuffers& B) {
    WChild c;
    c.code = code;
    if (code < 0) { c.lo = B.leaf_lo[~code]; c.hi = B.leaf_hi[~code]; }
    else { c.lo = B.node_lo[code]; c.hi = B.node_hi[code]; }
    return c;
}

__global__ void k_wide(BuildBuffers B, const int2* __restrict__ fin, int n_in, int2* fout, int* counters) {
    for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < n_in; it += gridDim.x * blockDim.x) {
        const int src = fin[it].x, dst = fin[it].y;
        WChild ch[BVH_W];
        int n = 2;
        ch[0] = make_child(B.left[src], B);
        ch[1] = make_child(B.right[src], B);
        while (n < BVH_W) {
            int best = -1;
            float ba = -1.0f;
            for (int c = 0; c < n; ++c) {
                if (is_open(ch[c].code, B.range, B.leaf_max)) {
                    const float a = half_area(ch[c].lo, ch[c].hi);
                    if (a > ba) { ba = a; best = c; }
                }
            }
            if (best < 0) break;
            const int code = ch[best].code;
            ch[best] = make_child(B.left[code], B);
            ch[n++] = make_child(B.right[code], B);
        }
        float3 lo[BVH_W], hi[BVH_W];
        int oc[BVH_W];
        for (int c = 0; c < BVH_W; ++c) {
            if (c >= n) {
                oc[c] = WIDE_EMPTY;
                continue;
            }
            lo[c] = f3(ch[c].lo.x, ch[c].lo.y, ch[c].lo.z);
            hi[c] = f3(ch[c].hi.x, ch[c].hi.y, ch[c].hi.z);
            const int code = ch[c].code;
            if (code < 0) {
                oc[c] = code;                                       // BVH2 leaf: ~slot (count 1)
            } else if (!is_open(code, B.range, B.leaf_max)) {
                const int2 r = B.range[code];
                oc[c] = ~(((r.y - r.x) << LEAF_SHIFT) | r.x);
            } else {
                const int slot = atomicAdd(&counters[1], 1);
                const int q = atomicAdd(&counters[0], 1);
                fout[q] = make_int2(code, slot);
                oc[c] = slot;
            }
        }
        node_write(B.nodes4 + NODE_F4 * (size_t)dst, lo, hi, oc);
    }
}

// ---------------------------------------------------------------- SAH-optimal 4-wide collapse
// Instead of opening the largest-area child until a node has 4 (k_wide), choose every BVH4 node's
// children by dynamic programming over the BVH2 (the wide-BVH collapse of Ylitie, Karras & Laine
// 2017, for width 4): with A = box surface area (hit probability), c_node the cost of a BVH4 node
// visit (4 box tests) and c_prim of a primitive test,
//   D(x, j) = least cost of covering x's subtree with at most j child slots of one wide node,
//   leaf:      D(x, j) = c_prim A(x)
//   internal:  open(x, j) = min_k D(l, k) + D(r, j - k),   C(x) = c_node A(x) + open(x, 4),
//              D(x, 1) = C(x),   D(x, j > 1) = min(C(x), open(x, j)),
// computed bottom-up (arrival flags, as k_refit); a wide node at x then takes the slots of
// open(x, 4) recursively (k_wide_dp).  choice[x]: best k of open(x, j) for j = 2, 3, 4 (2 bits
// each) and, for j = 2, 3, 4, whether x is opened (bit 6 + j - 2).
__device__ __forceinline__ void dp_child(int code, const BuildBuffers& B, const float* const* D, float c_prim, float d[4]) {
    if (code < 0) {
        const float c = c_prim * half_area(B.leaf_lo[~code], B.leaf_hi[~code]);
        d[0] = d[1] = d[2] = d[3] = c;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) d[j] = __ldcg(&D[j][code]);
    }
}

struct DpArrays {
    float* D[4];
    int* choice;
};

__global__ void k_collapse_dp(BuildBuffers B, int n, DpArrays X, float c_node, float c_prim) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        int p = B.parent_leaf[k];
        while (p >= 0) {
            __threadfence();
            if (atomicAdd(&B.flags[p], 1) == 0) break;    // first arrival: the sibling finishes p
            __threadfence();
            float dl[4], dr[4];
            dp_child(B.left[p], B, X.D, c_prim, dl);
            dp_child(B.right[p], B, X.D, c_prim, dr);
            float o[5];
            int kb[5];
#pragma unroll
            for (int j = 2; j <= 4; ++j) {
                o[j] = FLT_MAX;
                kb[j] = 1;
#pragma unroll
                for (int kk = 1; kk < j; ++kk) {
                    const float c = dl[kk - 1] + dr[j - kk - 1];
                    if (c < o[j]) { o[j] = c; kb[j] = kk; }
                }
            }
            const float C = c_node * half_area(B.node_lo[p], B.node_hi[p]) + o[4];
            int ch = kb[2] | (kb[3] << 2) | (kb[4] << 4);
            float d[4];
            d[0] = C;
#pragma unroll
            for (int j = 2; j <= 4; ++j) {
                const bool opened = o[j] < C;
                d[j - 1] = opened ? o[j] : C;
                ch |= (opened ? 1 : 0) << (6 + j - 2);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) __stcg(&X.D[j][p], d[j]);
            __stcg(&X.choice[p], ch);
            p = B.parent_int[p];
        }
    }
}

// BVH2 -> BVH4 by the DP choices: a wide node at BVH2 node src takes the slots of open(src, 4).
__global__ void k_wide_dp(BuildBuffers B, const int* __restrict__ choice, const int2* __restrict__ fin, int n_in, int2* fout,
                          int* counters) {
    for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < n_in; it += gridDim.x * blockDim.x) {
        const int src = fin[it].x, dst = fin[it].y;
        // expand (code, slots) pairs depth first; slots of a wide node: open(src, 4)
        int st_code[8], st_j[8], sp = 0;
        int codes[BVH_W], n = 0;
        const int c0 = choice[src], k4 = (c0 >> 4) & 3;
        st_code[sp] = B.right[src]; st_j[sp++] = 4 - k4;
        st_code[sp] = B.left[src]; st_j[sp++] = k4;
        while (sp > 0) {
            --sp;
            const int x = st_code[sp], j = st_j[sp];
            const int cx = x >= 0 ? choice[x] : 0;
            if (x < 0 || j == 1 || !((cx >> (6 + j - 2)) & 1)) {
                codes[n++] = x;                          // one slot: a leaf or a wide child node
            } else {
                const int kx = (cx >> (2 * (j - 2))) & 3;
                st_code[sp] = B.right[x]; st_j[sp++] = j - kx;
                st_code[sp] = B.left[x]; st_j[sp++] = kx;
            }
        }
        // the node's internal children get consecutive slots (one allocation), so siblings share
        // the cache lines at their boundaries
        int n_int = 0;
        for (int c = 0; c < n; ++c) n_int += codes[c] >= 0;
        int slot = 0, q = 0;
        if (n_int) {
            slot = atomicAdd(&counters[1], n_int);
            q = atomicAdd(&counters[0], n_int);
        }
        float3 lo[BVH_W], hi[BVH_W];
        int oc[BVH_W];
        for (int c = 0; c < BVH_W; ++c) {
            if (c >= n) {
                oc[c] = WIDE_EMPTY;
                continue;
            }
            const WChild w = make_child(codes[c], B);
            lo[c] = f3(w.lo.x, w.lo.y, w.lo.z);
            hi[c] = f3(w.hi.x, w.hi.y, w.hi.z);
            if (w.code < 0) {
                oc[c] = w.code;                                     // BVH2 leaf: ~slot (count 1)
            } else {
                fout[q++] = make_int2(w.code, slot);
                oc[c] = slot++;
            }
        }
        node_write(B.nodes4 + NODE_F4 * (size_t)dst, lo, hi, oc);
    }
}

// ---------------------------------------------------------------- SAH subtrees
// Every maximal LBVH subtree of at most SAH_T primitives (a contiguous Morton range [a, a + m) of
// leaf slots) is rebuilt top-down by binned SAH (3 axes x SAH_BINS bins, centroid binning).  The
// rebuild is level-synchronous over ALL subtrees at once: one warp per task (a node and its item
// range), bins in the warp's slice of shared memory, the split search as warp scans over the 32
// bins, a stable ballot partition; the children become the next level's tasks.  Node ids need no
// allocation: in a Karras LBVH the internal ids of a subtree over slots [a, a + m) are its root id
// and exactly [a + 1, a + m - 2], and the rule "left child = split position, right child = split
// position + 1" assigns that same set to ANY binary tree over the range (each internal node's id is
// its first or last position; two nodes could only share one if one were a leaf), so the subtree
// keeps its root and the nodes above it stay valid, and the result does not depend on the order
// tasks run in: the build is deterministic.  Runs before the treelet passes.  C4: node visits 16.2
// -> 15.5 per ray, bench +4.3 % (DESIGN.md §5 v21).
constexpr int SAH_T = 16384;
constexpr int SAH_BINS = 32;
constexpr int SAH_WARPS = 8;                 // warps (tasks) per CTA

__global__ void k_sah_roots(BuildBuffers B, int n, int* roots, int* n_roots) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n - 1; v += gridDim.x * blockDim.x) {
        const int2 r = B.range[v];
        if (r.y - r.x + 1 > SAH_T) continue;
        const int p = B.parent_int[v];
        if (p >= 0) {
            const int2 q = B.range[p];
            if (q.y - q.x + 1 <= SAH_T) continue;
        }
        roots[atomicAdd(n_roots, 1)] = v;
    }
}

// BVH2 depth budget of the SAH rebuild: a binned SAH split can peel off one primitive per level,
// so below (budget - ceil(log2 count)) levels a task is split at the median instead; the BVH2 (and
// therefore the BVH4 and its traversal stack, STACK_CAP) stays within SAH_MAX_DEPTH levels.
constexpr int SAH_MAX_DEPTH = 60;

__device__ __forceinline__ int ceil_log2(int n) { return n <= 1 ? 0 : 32 - __clz(n - 1); }

__device__ __forceinline__ int sah_bin(float c, float lo, float k) {
    return min(SAH_BINS - 1, max(0, (int)((c - lo) * k)));
}

// one warp per root: item slots [a, a + m) in order, the root's depth, the level-0 task
__global__ void k_sah_init(BuildBuffers B, const int* __restrict__ roots, int n_roots, int* idx, int4* tasks) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= n_roots) return;
    const int root = roots[w];
    const int2 rg = B.range[root];
    for (int k = rg.x + lane; k <= rg.y; k += 32) idx[k] = k;
    if (lane == 0) {
        int d0 = 0;
        for (int v = B.parent_int[root]; v >= 0; v = B.parent_int[v]) ++d0;
        tasks[w] = make_int4(rg.x, rg.y + 1, root, d0);
    }
}

struct SahWarpBins {
    int cnt[3][SAH_BINS];
    unsigned int lo[3][3][SAH_BINS], hi[3][3][SAH_BINS];    // [axis][component][bin], ordered floats
};
// Tasks of more than B.sah_big items (the top levels of a full SAH build) are split over many
// CTAs: every task's item range is cut into SAH_CHUNK-item chunks, one CTA per chunk, and the
// bounds, bins and left counts of a task are merged from its chunks with global atomics (min/max
// on ordered floats and integer adds: exact and order independent, so the tree is the one a single
// warp or CTA would build; tests/test_gpu_build.py).  Round 1 ran such a task on one 1024-thread
// CTA: 11 ms for the C4 root alone.
constexpr int SAH_CHUNK = 4096;              // items per CTA of a chunked task
constexpr int SAH_CTHR = 512;                  // threads per chunk CTA
constexpr int SAH_BIG_DEFAULT = 4096;        // tasks above this many items are chunked (env RT_SAH_BIG)

struct SahTaskAcc {                          // one chunked task's merged state (global memory)
    unsigned int v[12];                      // ordered floats: box lo/hi, centroid lo/hi
    SahWarpBins bins;
    int ax, bbin, nl, pad;
};

// per-level bookkeeping of the chunked tasks: task i's chunks are [cbase[i], cbase[i + 1]) in
// allocation order (a packed 64-bit counter hands out the task slot and its chunk range together)
struct SahChunked {
    int4* tasks;                             // (begin, end, node, depth)
    int* cbase;                              // first chunk of each task
    int* ctask;                              // chunk -> task
};

__device__ __forceinline__ void sah_bins_clear(SahWarpBins& S, int lane) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        S.cnt[q][lane] = 0;
#pragma unroll
        for (int e = 0; e < 3; ++e) { S.lo[q][e][lane] = 0xffffffffu; S.hi[q][e][lane] = 0u; }
    }
}

// bin one item (its leaf box) on every axis with extent
__device__ __forceinline__ void sah_bin_item(SahWarpBins& S, const BuildBuffers& B, int k, const float* v, const float* kq) {
    const float4 l4 = B.leaf_lo[k], h4 = B.leaf_hi[k];
    const float l[3] = {l4.x, l4.y, l4.z}, h[3] = {h4.x, h4.y, h4.z};
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        if (kq[q] == 0.0f) continue;
        const int b = sah_bin(0.5f * (l[q] + h[q]), v[6 + q], kq[q]);
        atomicAdd(&S.cnt[q][b], 1);
#pragma unroll
        for (int e = 0; e < 3; ++e) {
            atomicMin(&S.lo[q][e][b], f2ord(l[e]));
            atomicMax(&S.hi[q][e][b], f2ord(h[e]));
        }
    }
}

// Split search by one warp (lane = bin): SAH cost of splitting after every bin of every axis from
// prefix (bins <= lane) and suffix (bins > lane) scans; the lowest (cost, axis, bin) wins.
__device__ __forceinline__ void sah_split_search(const SahWarpBins& S, const float* kq, int lane, int& ax, int& bbin, int& nl) {
    const unsigned FULL = 0xffffffffu;
    unsigned long long best = ~0ull;                     // (cost bits << 32) | (axis * 32 + bin)
    int best_nl = 0;
    for (int q = 0; q < 3; ++q) {
        if (kq[q] == 0.0f) continue;
        const int c = S.cnt[q][lane];
        float pl[3], ph[3], sl[3], sh[3];
#pragma unroll
        for (int e = 0; e < 3; ++e) {
            pl[e] = sl[e] = c ? ord2f(S.lo[q][e][lane]) : FLT_MAX;
            ph[e] = sh[e] = c ? ord2f(S.hi[q][e][lane]) : -FLT_MAX;
        }
        int pc = c, sc = c;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int uc = __shfl_up_sync(FULL, pc, off), dc = __shfl_down_sync(FULL, sc, off);
            float ul[3], uh[3], dl[3], dh[3];
#pragma unroll
            for (int e = 0; e < 3; ++e) {
                ul[e] = __shfl_up_sync(FULL, pl[e], off); uh[e] = __shfl_up_sync(FULL, ph[e], off);
                dl[e] = __shfl_down_sync(FULL, sl[e], off); dh[e] = __shfl_down_sync(FULL, sh[e], off);
            }
            if (lane >= off) {
                pc += uc;
#pragma unroll
                for (int e = 0; e < 3; ++e) { pl[e] = fminf(pl[e], ul[e]); ph[e] = fmaxf(ph[e], uh[e]); }
            }
            if (lane + off < 32) {
                sc += dc;
#pragma unroll
                for (int e = 0; e < 3; ++e) { sl[e] = fminf(sl[e], dl[e]); sh[e] = fmaxf(sh[e], dh[e]); }
            }
        }
        const int rc = __shfl_down_sync(FULL, sc, 1);   // right side of a split after bin `lane`
        float rl[3], rh[3];
#pragma unroll
        for (int e = 0; e < 3; ++e) { rl[e] = __shfl_down_sync(FULL, sl[e], 1); rh[e] = __shfl_down_sync(FULL, sh[e], 1); }
        if (lane < SAH_BINS - 1 && pc > 0 && rc > 0) {
            const float cost = area3(f3(pl[0], pl[1], pl[2]), f3(ph[0], ph[1], ph[2])) * pc +
                               area3(f3(rl[0], rl[1], rl[2]), f3(rh[0], rh[1], rh[2])) * rc;
            const unsigned long long key = ((unsigned long long)__float_as_uint(cost) << 32) | (unsigned)(q * 32 + lane);
            if (key < best) { best = key; best_nl = pc; }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(FULL, best, off);
        const int onl = __shfl_xor_sync(FULL, best_nl, off);
        if (o < best) { best = o; best_nl = onl; }
    }
    if (best != ~0ull) {
        const unsigned id = (unsigned)(best & 0xffffffffu);
        ax = (int)(id >> 5);
        bbin = (int)(id & 31u);
        nl = best_nl;
    }
}

__device__ __forceinline__ bool sah_goes_left(const BuildBuffers& B, int k, int i, int begin, int ax, int bbin, int nl,
                                              const float* v, const float* kq) {
    if (ax < 0) return (i - begin) < nl;                 // median split in item order
    const float4 l4 = B.leaf_lo[k], h4 = B.leaf_hi[k];
    const float c = 0.5f * ((ax == 0 ? l4.x : ax == 1 ? l4.y : l4.z) + (ax == 0 ? h4.x : ax == 1 ? h4.y : h4.z));
    return sah_bin(c, v[6 + ax], kq[ax]) <= bbin;
}

// children of a split node (one thread): leaves get their slot codes, internal children their
// Karras ids and a task in the next level's list (chunked ones with their chunk range)
__device__ __forceinline__ void sah_children(const BuildBuffers& B, const int* idx, int begin, int end, int nl, int node,
                                             int depth, int4* next, int* n_next, SahChunked nb,
                                             unsigned long long* nb_ctr) {
    const int mid = begin + nl;
    int code[2];
    const int rb[2] = {begin, mid}, re[2] = {mid, end};
    for (int h = 0; h < 2; ++h) {
        if (re[h] - rb[h] == 1) {
            code[h] = ~idx[rb[h]];
            B.parent_leaf[idx[rb[h]]] = node;
        } else {
            code[h] = h == 0 ? mid - 1 : mid;            // Karras ids: split position / position + 1
            B.parent_int[code[h]] = node;
            B.range[code[h]] = make_int2(0, re[h] - rb[h] - 1);   // size only (leaf_max 1)
            const int4 t = make_int4(rb[h], re[h], code[h], depth + 1);
            if (re[h] - rb[h] > B.sah_big) {
                const int nch = (re[h] - rb[h] + SAH_CHUNK - 1) / SAH_CHUNK;
                const unsigned long long r = atomicAdd(nb_ctr, (1ull << 32) | (unsigned long long)nch);
                const int ti = (int)(r >> 32), c0 = (int)(r & 0xffffffffu);
                nb.tasks[ti] = t;
                nb.cbase[ti] = c0;
                for (int j = 0; j < nch; ++j) nb.ctask[c0 + j] = ti;
            } else {
                next[atomicAdd(n_next, 1)] = t;
            }
        }
    }
    B.left[node] = code[0];
    B.right[node] = code[1];
}

__device__ __forceinline__ void sah_kq(const float* v, float* kq) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const float ext = v[9 + q] - v[6 + q];
        kq[q] = ext > 0.0f ? SAH_BINS * (1.0f - 1e-6f) / ext : 0.0f;
    }
}

__device__ __forceinline__ void sah_bounds_item(const BuildBuffers& B, int k, float* v) {
    const float4 l4 = B.leaf_lo[k], h4 = B.leaf_hi[k];
    const float l[3] = {l4.x, l4.y, l4.z}, h[3] = {h4.x, h4.y, h4.z};
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const float c = 0.5f * (l[q] + h[q]);
        v[q] = fminf(v[q], l[q]); v[3 + q] = fmaxf(v[3 + q], h[q]);
        v[6 + q] = fminf(v[6 + q], c); v[9 + q] = fmaxf(v[9 + q], c);
    }
}

__device__ __forceinline__ void sah_bounds_init(float* v) {
#pragma unroll
    for (int q = 0; q < 3; ++q) { v[q] = FLT_MAX; v[3 + q] = -FLT_MAX; v[6 + q] = FLT_MAX; v[9 + q] = -FLT_MAX; }
}

__device__ __forceinline__ void sah_bounds_warp(float* v) {
#pragma unroll
    for (int q = 0; q < 12; ++q) {
        const bool mx = (q >= 3 && q < 6) || q >= 9;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const float o = __shfl_xor_sync(0xffffffffu, v[q], off);
            v[q] = mx ? fmaxf(v[q], o) : fminf(v[q], o);
        }
    }
}

// One level, tasks of <= B.sah_big items: task (begin, end, node, depth) per warp over idx[begin, end).
__global__ void __launch_bounds__(32 * SAH_WARPS) k_sah_level(BuildBuffers B, const int4* __restrict__ tasks,
                                                              int n_tasks, int4* next, int* n_next, SahChunked nb,
                                                              unsigned long long* nb_ctr, int* idx, int* tmp) {
    __shared__ SahWarpBins bins[SAH_WARPS];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int w = blockIdx.x * SAH_WARPS + wl;
    if (w >= n_tasks) return;
    const unsigned FULL = 0xffffffffu;
    const int4 t = tasks[w];
    const int begin = t.x, end = t.y, node = t.z, depth = t.w, cnt = end - begin;
    const bool median = depth + ceil_log2(cnt) >= SAH_MAX_DEPTH;   // depth budget: balanced below
    float v[12];                                         // node box and centroid bounds
    sah_bounds_init(v);
    for (int i = begin + lane; i < end; i += 32) sah_bounds_item(B, idx[i], v);
    sah_bounds_warp(v);
    if (lane == 0) {
        B.node_lo[node] = make_float4(v[0], v[1], v[2], 0.f);
        B.node_hi[node] = make_float4(v[3], v[4], v[5], 0.f);
    }
    float kq[3];
    sah_kq(v, kq);
    int ax = -1, nl = cnt / 2, bbin = 0;                 // no split found: halve the list
    if (cnt > 2 && !median) {
        SahWarpBins& S = bins[wl];
        sah_bins_clear(S, lane);
        __syncwarp();
        for (int i = begin + lane; i < end; i += 32) sah_bin_item(S, B, idx[i], v, kq);
        __syncwarp();
        sah_split_search(S, kq, lane, ax, bbin, nl);
    }
    int lbase = 0, rbase = 0;                            // stable partition into tmp, then back
    for (int c0 = begin; c0 < end; c0 += 32) {
        const int i = c0 + lane;
        const int k = i < end ? idx[i] : 0;
        const bool left = i < end && sah_goes_left(B, k, i, begin, ax, bbin, nl, v, kq);
        const unsigned bal = __ballot_sync(FULL, left);
        const int lrank = __popc(bal & ((1u << lane) - 1u));
        if (i < end) tmp[left ? begin + lbase + lrank : begin + nl + rbase + (lane - lrank)] = k;
        lbase += __popc(bal);
        rbase += min(32, end - c0) - __popc(bal);
    }
    __syncwarp();
    for (int i = begin + lane; i < end; i += 32) idx[i] = tmp[i];
    __syncwarp();
    if (lane == 0) sah_children(B, idx, begin, end, nl, node, depth, next, n_next, nb, nb_ctr);
}

// ---- chunked tasks (> B.sah_big items): one level = init, bounds, bins, split, count, scatter,
// copy back + children; every kernel but init / split runs one CTA per chunk
__device__ __forceinline__ void chunk_range(const SahChunked& T, int chunk, int& task, int4& t, int& lo, int& hi) {
    task = T.ctask[chunk];
    t = T.tasks[task];
    lo = t.x + (chunk - T.cbase[task]) * SAH_CHUNK;
    hi = min(t.y, lo + SAH_CHUNK);
}

__device__ __forceinline__ bool chunk_median(const int4& t) { return t.w + ceil_log2(t.y - t.x) >= SAH_MAX_DEPTH; }

__global__ void k_sah_chunk_init(SahTaskAcc* acc, int n_tasks) {
    constexpr int WORDS = sizeof(SahTaskAcc) / 4;
    unsigned int* a = reinterpret_cast<unsigned int*>(acc + blockIdx.x);
    if (blockIdx.x >= n_tasks) return;
    for (int e = threadIdx.x; e < WORDS; e += blockDim.x) {
        unsigned int x = 0u;                                     // counts, maxima, split fields
        if (e < 12) x = (e < 3 || (e >= 6 && e < 9)) ? 0xffffffffu : 0u;
        else if (e >= 12 + 3 * SAH_BINS && e < 12 + 12 * SAH_BINS) x = 0xffffffffu;   // bin minima
        a[e] = x;
    }
}

// CTA-wide reduction of v[12] (min for box/centroid lo, max for hi) into acc[task].v
__global__ void __launch_bounds__(SAH_CTHR) k_sah_chunk_bounds(BuildBuffers B, SahChunked T, SahTaskAcc* acc,
                                                              const int* __restrict__ idx) {
    __shared__ float red[SAH_CTHR / 32][12];
    int task, lo, hi;
    int4 t;
    chunk_range(T, blockIdx.x, task, t, lo, hi);
    float v[12];
    sah_bounds_init(v);
    for (int i = lo + threadIdx.x; i < hi; i += SAH_CTHR) sah_bounds_item(B, idx[i], v);
    sah_bounds_warp(v);
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    if (lane == 0)
        for (int q = 0; q < 12; ++q) red[wl][q] = v[q];
    __syncthreads();
    if (threadIdx.x < 12) {
        const int q = threadIdx.x;
        const bool mx = (q >= 3 && q < 6) || q >= 9;
        float x = red[0][q];
        for (int w = 1; w < SAH_CTHR / 32; ++w) x = mx ? fmaxf(x, red[w][q]) : fminf(x, red[w][q]);
        if (mx) atomicMax(&acc[task].v[q], f2ord(x));
        else atomicMin(&acc[task].v[q], f2ord(x));
    }
}

__device__ __forceinline__ void acc_bounds(const SahTaskAcc& A, float* v) {
#pragma unroll
    for (int q = 0; q < 12; ++q) v[q] = ord2f(A.v[q]);
}

// per-warp shared bins, merged per CTA, then into acc[task].bins with global atomics
__global__ void __launch_bounds__(SAH_CTHR) k_sah_chunk_bin(BuildBuffers B, SahChunked T, SahTaskAcc* acc,
                                                           const int* __restrict__ idx) {
    extern __shared__ SahWarpBins cb[];                  // [SAH_CTHR / 32]
    int task, lo, hi;
    int4 t;
    chunk_range(T, blockIdx.x, task, t, lo, hi);
    if (t.y - t.x <= 2 || chunk_median(t)) return;
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    float v[12], kq[3];
    acc_bounds(acc[task], v);
    sah_kq(v, kq);
    sah_bins_clear(cb[wl], lane);
    __syncthreads();
    for (int i = lo + threadIdx.x; i < hi; i += SAH_CTHR) sah_bin_item(cb[wl], B, idx[i], v, kq);
    __syncthreads();
    constexpr int ENTRIES = sizeof(SahWarpBins) / 4;
    const unsigned* base = reinterpret_cast<const unsigned*>(cb);
    unsigned* dst = reinterpret_cast<unsigned*>(&acc[task].bins);
    for (int e = threadIdx.x; e < ENTRIES; e += SAH_CTHR) {
        const bool is_cnt = e < 3 * SAH_BINS, is_lo = !is_cnt && e < 3 * SAH_BINS + 9 * SAH_BINS;
        unsigned x = base[e];
        for (int w = 1; w < SAH_CTHR / 32; ++w) {
            const unsigned y = base[w * ENTRIES + e];
            x = is_cnt ? x + y : (is_lo ? min(x, y) : max(x, y));
        }
        if (is_cnt) { if (x) atomicAdd(&dst[e], x); }
        else if (is_lo) { if (x != 0xffffffffu) atomicMin(&dst[e], x); }
        else if (x) atomicMax(&dst[e], x);
    }
}

// one warp per task: node box, then the split (the same search as a warp task)
__global__ void k_sah_chunk_split(BuildBuffers B, SahChunked T, SahTaskAcc* acc, int n_tasks) {
    __shared__ SahWarpBins S;
    const int task = blockIdx.x, lane = threadIdx.x;
    if (task >= n_tasks) return;
    const int4 t = T.tasks[task];
    const int cnt = t.y - t.x;
    float v[12], kq[3];
    acc_bounds(acc[task], v);
    if (lane == 0) {
        B.node_lo[t.z] = make_float4(v[0], v[1], v[2], 0.f);
        B.node_hi[t.z] = make_float4(v[3], v[4], v[5], 0.f);
    }
    sah_kq(v, kq);
    int ax = -1, nl = cnt / 2, bbin = 0;
    if (cnt > 2 && !chunk_median(t)) {
        const unsigned* src = reinterpret_cast<const unsigned*>(&acc[task].bins);
        unsigned* dst = reinterpret_cast<unsigned*>(&S);
        for (int e = lane; e < (int)(sizeof(SahWarpBins) / 4); e += 32) dst[e] = src[e];
        __syncwarp();
        sah_split_search(S, kq, lane, ax, bbin, nl);
    }
    if (lane == 0) { acc[task].ax = ax; acc[task].bbin = bbin; acc[task].nl = nl; }
}

// left items of every chunk
__global__ void __launch_bounds__(SAH_CTHR) k_sah_chunk_count(BuildBuffers B, SahChunked T, const SahTaskAcc* acc,
                                                             const int* __restrict__ idx, int* cleft) {
    __shared__ int wsum[SAH_CTHR / 32];
    int task, lo, hi;
    int4 t;
    chunk_range(T, blockIdx.x, task, t, lo, hi);
    const SahTaskAcc& A = acc[task];
    float v[12], kq[3];
    acc_bounds(A, v);
    sah_kq(v, kq);
    int c = 0;
    for (int i = lo + threadIdx.x; i < hi; i += SAH_CTHR) c += sah_goes_left(B, idx[i], i, t.x, A.ax, A.bbin, A.nl, v, kq);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int s2 = 0;
        for (int w = 0; w < SAH_CTHR / 32; ++w) s2 += wsum[w];
        cleft[blockIdx.x] = s2;
    }
}

// stable partition of the chunk into tmp: left items after the left items of the task's earlier
// chunks, right items after theirs
__global__ void __launch_bounds__(SAH_CTHR) k_sah_chunk_scatter(BuildBuffers B, SahChunked T, const SahTaskAcc* acc,
                                                               const int* __restrict__ idx, const int* __restrict__ cleft,
                                                               int* tmp) {
    __shared__ int wcnt[SAH_CTHR / 32 + 1];
    __shared__ int lbase_s;
    int task, lo, hi;
    int4 t;
    chunk_range(T, blockIdx.x, task, t, lo, hi);
    const SahTaskAcc& A = acc[task];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    if (wl == 0) {                                        // left items in this task's earlier chunks
        int s2 = 0;
        for (int c = T.cbase[task] + lane; c < (int)blockIdx.x; c += 32) s2 += cleft[c];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, off);
        if (lane == 0) lbase_s = s2;
    }
    float v[12], kq[3];
    acc_bounds(A, v);
    sah_kq(v, kq);
    __syncthreads();
    int lbase = lbase_s, rbase = (lo - t.x) - lbase_s;
    for (int c0 = lo; c0 < hi; c0 += SAH_CTHR) {
        const int i = c0 + threadIdx.x;
        const int k = i < hi ? idx[i] : 0;
        const bool left = i < hi && sah_goes_left(B, k, i, t.x, A.ax, A.bbin, A.nl, v, kq);
        const unsigned bal = __ballot_sync(0xffffffffu, left);
        if (lane == 0) wcnt[wl] = __popc(bal);
        __syncthreads();
        if (threadIdx.x == 0) {
            int acc2 = 0;
            for (int w = 0; w < SAH_CTHR / 32; ++w) { const int x = wcnt[w]; wcnt[w] = acc2; acc2 += x; }
            wcnt[SAH_CTHR / 32] = acc2;
        }
        __syncthreads();
        const int lrank = wcnt[wl] + __popc(bal & ((1u << lane) - 1u));
        const int chunk_l = wcnt[SAH_CTHR / 32];
        if (i < hi) tmp[left ? t.x + lbase + lrank : t.x + A.nl + rbase + (i - c0 - lrank)] = k;
        lbase += chunk_l;
        rbase += min(SAH_CTHR, hi - c0) - chunk_l;
        __syncthreads();
    }
}

// partitioned order back into idx; the task's first chunk emits its children (reading tmp, which
// holds the same order)
__global__ void __launch_bounds__(SAH_CTHR) k_sah_chunk_finish(BuildBuffers B, SahChunked T, const SahTaskAcc* acc,
                                                              int* idx, const int* __restrict__ tmp, int4* next,
                                                              int* n_next, SahChunked nb, unsigned long long* nb_ctr) {
    int task, lo, hi;
    int4 t;
    chunk_range(T, blockIdx.x, task, t, lo, hi);
    for (int i = lo + threadIdx.x; i < hi; i += SAH_CTHR) idx[i] = tmp[i];
    if (threadIdx.x == 0 && (int)blockIdx.x == T.cbase[task])
        sah_children(B, tmp, t.x, t.y, acc[task].nl, t.z, t.w, next, n_next, nb, nb_ctr);
}

// the whole tree (Karras root 0, slots [0, n)) as one chunked task: identity item order, every
// chunk mapped to task 0 (full SAH build of n > B.sah_big items)
__global__ void k_sah_chunk_seed(SahChunked T, int* idx, int n, int depth0) {
    const int nch = (n + SAH_CHUNK - 1) / SAH_CHUNK;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        idx[j] = j;
        if (j < nch) T.ctask[j] = 0;
        if (j == 0) {
            T.tasks[0] = make_int4(0, n, 0, depth0);
            T.cbase[0] = 0;
        }
    }
}

// leaf-order records and leaf AABBs (slot k = sorted position k)
__global__ void k_gather_prims(BuildBuffers B, int n, const uint32_t* __restrict__ order, float4* slo, float4* shi) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const uint32_t s = order[k];
        B.prims[3 * k] = B.prims_unsorted[3 * s];
        B.prims[3 * k + 1] = B.prims_unsorted[3 * s + 1];
        B.prims[3 * k + 2] = B.prims_unsorted[3 * s + 2];
        slo[k] = B.aabb_lo[s];
        shi[k] = B.aabb_hi[s];
    }
}

// ---------------------------------------------------------------- refit (NEXT-3: moving vertices)
// New vertex positions -> leaf-order triangle records (v0, e1, e2); topology and leaf order kept.
__global__ void k_update_prims(float4* prims, const int* __restrict__ prim_orig, int n, int n_spheres,
                               const uint32_t* __restrict__ tri_idx, const float* __restrict__ vtx) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int o = prim_orig[k];
        if (o < n_spheres) continue;
        const int j = o - n_spheres;
        const uint32_t a = tri_idx[3 * j], b = tri_idx[3 * j + 1], c = tri_idx[3 * j + 2];
        const float3 v0 = f3(vtx[3 * a], vtx[3 * a + 1], vtx[3 * a + 2]);
        const float3 v1 = f3(vtx[3 * b], vtx[3 * b + 1], vtx[3 * b + 2]);
        const float3 v2 = f3(vtx[3 * c], vtx[3 * c + 1], vtx[3 * c + 2]);
        const float4 r0 = prims[3 * k], r1 = prims[3 * k + 1];
        prims[3 * k] = make_float4(v0.x, v0.y, v0.z, r0.w);
        prims[3 * k + 1] = make_float4(v1.x - v0.x, v1.y - v0.y, v1.z - v0.z, r1.w);
        prims[3 * k + 2] = make_float4(v2.x - v0.x, v2.y - v0.y, v2.z - v0.z, 0.f);
    }
}

__device__ __forceinline__ void prim_box(int k, const int* __restrict__ prim_orig, int n_spheres,
                                         const float4* __restrict__ spheres, const uint32_t* __restrict__ tri_idx,
                                         const float* __restrict__ vtx, float3& lo, float3& hi) {
    const int o = prim_orig[k];
    if (o < n_spheres) {
        const float4 s = spheres[o];
        lo = f3(__fsub_rd(s.x, s.w), __fsub_rd(s.y, s.w), __fsub_rd(s.z, s.w));
        hi = f3(__fadd_ru(s.x, s.w), __fadd_ru(s.y, s.w), __fadd_ru(s.z, s.w));
        return;
    }
    const int j = o - n_spheres;
    const uint32_t a = tri_idx[3 * j], b = tri_idx[3 * j + 1], c = tri_idx[3 * j + 2];
    lo = f3(fminf(vtx[3 * a], fminf(vtx[3 * b], vtx[3 * c])), fminf(vtx[3 * a + 1], fminf(vtx[3 * b + 1], vtx[3 * c + 1])),
            fminf(vtx[3 * a + 2], fminf(vtx[3 * b + 2], vtx[3 * c + 2])));
    hi = f3(fmaxf(vtx[3 * a], fmaxf(vtx[3 * b], vtx[3 * c])), fmaxf(vtx[3 * a + 1], fmaxf(vtx[3 * b + 1], vtx[3 * c + 1])),
            fmaxf(vtx[3 * a + 2], fmaxf(vtx[3 * b + 2], vtx[3 * c + 2])));
}

// Bottom-up refit of one BVH4 level (nodes [begin, end)); deeper levels are already refit, and
// empty slots are skipped and rewritten as empty.
__global__ void k_refit4(float4* nodes, int begin, int end, const int* __restrict__ prim_orig, int n_spheres,
                         const float4* __restrict__ spheres, const uint32_t* __restrict__ tri_idx,
                         const float* __restrict__ vtx) {
    for (int i = begin + blockIdx.x * blockDim.x + threadIdx.x; i < end; i += gridDim.x * blockDim.x) {
        float4* q = nodes + NODE_F4 * (size_t)i;
        float3 L[BVH_W], Hh[BVH_W];
        int codes[BVH_W];
        for (int c = 0; c < BVH_W; ++c) {
            float3 l = f3(1e30f, 1e30f, 1e30f), h = f3(-1e30f, -1e30f, -1e30f);
            const int code = node_code(q, c);
            codes[c] = code;
            if (code == WIDE_EMPTY) {
            } else if (code < 0) {
                const int enc = ~code;
                const int first = enc & ((1 << LEAF_SHIFT) - 1), last = first + (enc >> LEAF_SHIFT);
                for (int k = first; k <= last; ++k) {
                    float3 pl, ph;
                    prim_box(k, prim_orig, n_spheres, spheres, tri_idx, vtx, pl, ph);
                    l = f3(fminf(l.x, pl.x), fminf(l.y, pl.y), fminf(l.z, pl.z));
                    h = f3(fmaxf(h.x, ph.x), fmaxf(h.y, ph.y), fmaxf(h.z, ph.z));
                }
            } else {
                const float4* r = nodes + NODE_F4 * (size_t)code;
                for (int k = 0; k < BVH_W; ++k) {
                    if (node_code(r, k) == WIDE_EMPTY) continue;
                    float3 bl, bh;
                    node_child_box(r, k, bl, bh);
                    l = f3(fminf(l.x, bl.x), fminf(l.y, bl.y), fminf(l.z, bl.z));
                    h = f3(fmaxf(h.x, bh.x), fmaxf(h.y, bh.y), fmaxf(h.z, bh.z));
                }
            }
            L[c] = l;
            Hh[c] = h;
        }
        node_write(q, L, Hh, codes);
    }
}

}  // namespace rtb

using namespace rtb;

size_t rtb_sort_hist_entries(int n) { return 256u * (size_t)((n + SORT_TILE - 1) / SORT_TILE); }

static int grid_for(int n, int block = 256) {
    const int g = (n + block - 1) / block;
    return g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g);
}

cudaError_t rtb_build_bvh(const BuildBuffers& Bc, cudaStream_t st, int* root, int* n_nodes4, int* depth4,
                          int* level_start) {
    BuildBuffers B = Bc;
    const int n = B.n_spheres + B.n_tris;
    if (n == 0) return cudaSuccess;
    k_prim_setup<<<grid_for(n), 256, 0, st>>>(B);
    if (n == 1) {
        cudaMemcpyAsync(B.prims, B.prims_unsorted, 3 * sizeof(float4), cudaMemcpyDeviceToDevice, st);
        cudaMemsetAsync(B.prim_orig, 0, sizeof(int), st);
        *root = ~0;
        *n_nodes4 = 0;
        *depth4 = 0;
        return cudaGetLastError();
    }
    k_bounds_init<<<1, 32, 0, st>>>(B.bounds);
    k_bounds<<<grid_for(n), 256, 0, st>>>(B.centroid, n, B.bounds);
    k_morton<<<grid_for(n), 256, 0, st>>>(B.centroid, n, B.bounds, B.keys[0], B.vals[0]);
    const int nb = (n + SORT_TILE - 1) / SORT_TILE;
    int cur = 0;
    for (int shift = 0; shift < 30; shift += 8) {
        k_radix_hist<<<nb, SORT_THREADS, 0, st>>>(B.keys[cur], n, shift, B.hist, nb);
        k_scan_single<<<1, 1024, 0, st>>>(B.hist, 256 * nb);
        k_radix_scatter<<<nb, SORT_THREADS, 0, st>>>(B.keys[cur], B.vals[cur], B.keys[cur ^ 1], B.vals[cur ^ 1], n,
                                                     shift, B.hist, nb);
        cur ^= 1;
    }
    float4* slo = B.leaf_lo;
    float4* shi = B.leaf_hi;
    k_gather_prims<<<grid_for(n), 256, 0, st>>>(B, n, B.vals[cur], slo, shi);
    cudaMemcpyAsync(B.prim_orig, B.vals[cur], sizeof(int) * n, cudaMemcpyDeviceToDevice, st);
    k_karras<<<grid_for(n - 1), 256, 0, st>>>(B.keys[cur], n, B.left, B.right, B.parent_int, B.parent_leaf, B.range);
    cudaMemsetAsync(B.flags, 0, sizeof(int) * (n - 1), st);
    k_refit<<<grid_for(n), 256, 0, st>>>(B, n, slo, shi);
    // SAH subtrees, then treelet restructuring passes (SAH); leaf collapse by sorted range needs
    // the original Morton topology, so both run only without it
    if (B.leaf_max == 1 && n > 2 && B.sah_subtrees) {
        int* roots = B.frontier[0] ? reinterpret_cast<int*>(B.frontier[0]) : nullptr;   // scratch [N] int2
        int* n_roots = B.wide_counters;
        int h_roots = 0;
        if (B.sah_subtrees == 2) {                       // full SAH: the whole tree is one subtree
            cudaMemsetAsync(roots, 0, sizeof(int), st);  // Karras root 0, slots [0, n)
            h_roots = 1;
        } else {
            cudaMemsetAsync(n_roots, 0, sizeof(int), st);
            k_sah_roots<<<grid_for(n - 1), 256, 0, st>>>(B, n, roots, n_roots);
            cudaMemcpyAsync(&h_roots, n_roots, sizeof(int), cudaMemcpyDeviceToHost, st);
        }
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return e;
        // scratch: the sort keys are free once the leaves are gathered and the hierarchy built
        // (item order idx / tmp); the level task lists borrow frontier[1] and the BVH4 staging
        // (each >= N/2 int4, unused until k_wide)
        if (h_roots > 0) {
            int* idx = reinterpret_cast<int*>(B.keys[0]);
            int* tmp = reinterpret_cast<int*>(B.keys[1]);
            // task lists: warp tasks of the current and the next level in frontier[1] / the BVH4
            // staging (each >= N/2 int4, unused until k_wide); behind the latter the chunked
            // tasks' lists, chunk maps and merged state (sized for n / sah_big tasks a level)
            int4* base4 = reinterpret_cast<int4*>(B.nodes4);
            int4* tl[2] = {reinterpret_cast<int4*>(B.frontier[1]), base4};
            int* n_next = B.wide_counters + 1;
            unsigned long long* nb_ctr = reinterpret_cast<unsigned long long*>(B.wide_counters + 2);
            SahChunked tc[2] = {};
            SahTaskAcc* acc = nullptr;
            int* cleft = nullptr;
            if (n > B.sah_big) {
                const size_t max_t = (size_t)n / B.sah_big + 2, max_c = (size_t)n / SAH_CHUNK + max_t + 1;
                char* p = reinterpret_cast<char*>(base4 + (n / 2 + 1));
                auto carve = [&](size_t bytes) { char* q = p; p += (bytes + 255) & ~size_t(255); return q; };
                for (int k = 0; k < 2; ++k) {
                    tc[k].tasks = reinterpret_cast<int4*>(carve(max_t * sizeof(int4)));
                    tc[k].cbase = reinterpret_cast<int*>(carve(max_t * sizeof(int)));
                    tc[k].ctask = reinterpret_cast<int*>(carve(max_c * sizeof(int)));
                }
                cleft = reinterpret_cast<int*>(carve(max_c * sizeof(int)));
                acc = reinterpret_cast<SahTaskAcc*>(carve(max_t * sizeof(SahTaskAcc)));
                // the whole carve must stay inside the BVH4 staging (16 * NODE_F4 * (n - 1) bytes)
                if (p > reinterpret_cast<char*>(B.nodes4) + 16 * (size_t)NODE_F4 * (size_t)(n - 1))
                    return cudaErrorInvalidValue;
            }
            static_assert(sizeof(SahWarpBins) * (SAH_CTHR / 32) <= 48 * 1024, "chunk bins fit the default dynamic smem");
            int n_small = 0, n_big = 0, n_chunks = 0;
            if (B.sah_subtrees == 2 && n > B.sah_big) {
                k_sah_chunk_seed<<<grid_for(n), 256, 0, st>>>(tc[0], idx, n, 0);
                n_big = 1;
                n_chunks = (n + SAH_CHUNK - 1) / SAH_CHUNK;
            } else {
                k_sah_init<<<(h_roots * 32 + 255) / 256, 256, 0, st>>>(B, roots, h_roots, idx, tl[0]);
                n_small = h_roots;
            }
            int cur = 0;
            while (n_small + n_big > 0) {
                cudaMemsetAsync(B.wide_counters + 1, 0, 3 * sizeof(int), st);   // n_next + nb_ctr
                const SahChunked& T = tc[cur];
                const SahChunked& N2 = tc[cur ^ 1];
                if (n_big) {
                    k_sah_chunk_init<<<n_big, 256, 0, st>>>(acc, n_big);
                    k_sah_chunk_bounds<<<n_chunks, SAH_CTHR, 0, st>>>(B, T, acc, idx);
                    k_sah_chunk_bin<<<n_chunks, SAH_CTHR, sizeof(SahWarpBins) * (SAH_CTHR / 32), st>>>(B, T, acc, idx);
                    k_sah_chunk_split<<<n_big, 32, 0, st>>>(B, T, acc, n_big);
                    k_sah_chunk_count<<<n_chunks, SAH_CTHR, 0, st>>>(B, T, acc, idx, cleft);
                    k_sah_chunk_scatter<<<n_chunks, SAH_CTHR, 0, st>>>(B, T, acc, idx, cleft, tmp);
                    k_sah_chunk_finish<<<n_chunks, SAH_CTHR, 0, st>>>(B, T, acc, idx, tmp, tl[cur ^ 1], n_next, N2, nb_ctr);
                }
                if (n_small)
                    k_sah_level<<<(n_small + SAH_WARPS - 1) / SAH_WARPS, 32 * SAH_WARPS, 0, st>>>(
                        B, tl[cur], n_small, tl[cur ^ 1], n_next, N2, nb_ctr, idx, tmp);
                int h[3];
                cudaMemcpyAsync(h, B.wide_counters + 1, 3 * sizeof(int), cudaMemcpyDeviceToHost, st);
                e = cudaStreamSynchronize(st);
                if (e != cudaSuccess) return e;
                unsigned long long ctr;
                memcpy(&ctr, h + 1, sizeof ctr);
                n_small = h[0];
                n_big = (int)(ctr >> 32);
                n_chunks = (int)(ctr & 0xffffffffu);
                cur ^= 1;
            }
        }
    }
    if (B.leaf_max == 1) {
        for (int pass = 0; pass < B.treelet_passes; ++pass) {
            cudaMemsetAsync(B.flags, 0, sizeof(int) * (n - 1), st);
            k_treelets<<<grid_for(n), 256, 0, st>>>(B, n);
        }
    }
    // root: a leaf if the whole scene fits one leaf, else BVH4 node 0 from BVH2 node 0
    if (n <= B.leaf_max) {
        *root = ~(((n - 1) << LEAF_SHIFT) | 0);
        *n_nodes4 = 0;
        *depth4 = 0;
        return cudaGetLastError();
    }
    // SAH-optimal collapse (leaf_max 1): DP tables in the sort scratch (free after the SAH build)
    const bool dp = B.leaf_max == 1 && B.collapse_dp;
    DpArrays dpx{};
    if (dp) {
        dpx.D[0] = reinterpret_cast<float*>(B.keys[0]);
        dpx.D[1] = reinterpret_cast<float*>(B.keys[1]);
        dpx.D[2] = reinterpret_cast<float*>(B.vals[0]);
        dpx.D[3] = reinterpret_cast<float*>(B.vals[1]);
        dpx.choice = B.count;
        cudaMemsetAsync(B.flags, 0, sizeof(int) * (n - 1), st);
        k_collapse_dp<<<grid_for(n), 256, 0, st>>>(B, n, dpx, 1.0f, B.collapse_cprim);
    }
    int2 first = make_int2(0, 0);
    int h_counters[2] = {0, 1};
    if (level_start) { level_start[0] = 0; level_start[1] = 1; }
    cudaMemcpyAsync(B.frontier[0], &first, sizeof(int2), cudaMemcpyHostToDevice, st);
    int n_in = 1, levels = 0, cur_f = 0;
    while (n_in > 0) {
        h_counters[0] = 0;
        cudaMemcpyAsync(B.wide_counters, h_counters, sizeof(int), cudaMemcpyHostToDevice, st);
        if (levels == 0) cudaMemcpyAsync(B.wide_counters + 1, h_counters + 1, sizeof(int), cudaMemcpyHostToDevice, st);
        if (dp)
            k_wide_dp<<<grid_for(n_in), 256, 0, st>>>(B, dpx.choice, B.frontier[cur_f], n_in, B.frontier[cur_f ^ 1],
                                                      B.wide_counters);
        else
            k_wide<<<grid_for(n_in), 256, 0, st>>>(B, B.frontier[cur_f], n_in, B.frontier[cur_f ^ 1], B.wide_counters);
        cudaError_t e = cudaMemcpyAsync(h_counters, B.wide_counters, 2 * sizeof(int), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return e;
        n_in = h_counters[0];
        cur_f ^= 1;
        ++levels;
        if (level_start && levels + 1 <= 65) level_start[levels + 1] = h_counters[1];
    }
    *root = 0;
    *n_nodes4 = h_counters[1];
    *depth4 = levels;
    return cudaGetLastError();
}

cudaError_t rtb_refit_bvh(float4* prims, float4* nodes4, const int* prim_orig, int n, int n_spheres,
                          const float4* spheres, const uint32_t* tri_idx, const float* vtx,
                          const int* level_start, int levels, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_update_prims<<<grid_for(n), 256, 0, st>>>(prims, prim_orig, n, n_spheres, tri_idx, vtx);
    for (int L = levels - 1; L >= 0; --L) {
        const int b = level_start[L], e = level_start[L + 1];
        if (e > b) k_refit4<<<grid_for(e - b), 256, 0, st>>>(nodes4, b, e, prim_orig, n_spheres, spheres, tri_idx, vtx);
    }
    return cudaGetLastError();
}
