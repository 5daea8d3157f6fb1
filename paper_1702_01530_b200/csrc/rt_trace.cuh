// rt_trace.cuh -- device code shared by the trace kernels: work-item -> pixel mapping, output
// packing, primitive tests, 4-wide BVH traversal (nearest hit and any hit).
#pragma once
#include "rt_device.cuh"
#include "rt_internal.h"

namespace rtb {

constexpr int RT_BLOCK = 64;      // threads per trace CTA (stack stride); small CTAs free their slots as soon as
                                  // their 2 warps finish, so a next frame in flight fills the SM sooner
#ifndef RT_SMEM_STACK_X
constexpr int RT_SMEM_STACK = 16; // traversal-stack entries kept in shared memory; deeper ones in local
#else
constexpr int RT_SMEM_STACK = RT_SMEM_STACK_X;
#endif
constexpr int RT_OCC_LIGHTS = 4;  // lights with a last-occluder hint slot (light j uses slot j; others none)

// Per-thread traversal stack: the first RT_SMEM_STACK entries live in shared memory laid out
// [entry][thread] (conflict-free), deeper entries in thread-local memory (L1-cached).  Keeping the
// shared part short leaves most of the 228 KB L1/shared array to cache BVH nodes.
//
// The stack pointer is the byte offset of the next memory entry in the CTA's stack array:
// sp = i * E + 4 * tid for logical memory depth i (E = RT_BLOCK * 4 bytes per entry row; 4 * tid
// < E, so i = sp / E).  One loop-carried register is depth, emptiness test (sp < E, an immediate
// compare) and STS/LDS offset; the array's shared-window address `base` is the same for every
// thread and sits in a uniform register (STS [R + UR]).  It is pinned there through a volatile
// move: plain __cvta_generic_to_shared values are rematerialised by ptxas at every use from
// S2R SR_CgaCtaId (+ SR_TID.X for a per-thread base, as in round 1), which put S2R latencies in
// front of every push and refill load.
constexpr uint32_t STK_E = RT_BLOCK * 4u;   // bytes per stack entry row

// A value ptxas must keep (or spill) rather than rematerialise at every use: the result of a
// volatile move cannot be recomputed.
__device__ __forceinline__ uint32_t pin_reg(uint32_t a) {
    uint32_t r;
    asm volatile("mov.u32 %0, %1;" : "=r"(r) : "r"(a));
    return r;
}

struct TravStack {
    uint32_t base;   // shared-window byte address of the CTA's stack array (uniform)
    int* l;          // local part: logical entry i >= RT_SMEM_STACK at l[i - RT_SMEM_STACK]
    __device__ __forceinline__ static uint32_t pin(uint32_t a) { return pin_reg(a); }
    __device__ __forceinline__ static uint32_t empty() { return 4u * threadIdx.x; }
    __device__ __forceinline__ static bool nonempty(uint32_t a) { return a >= STK_E; }
    // true when entries a and a + E both lie in the shared part
    __device__ __forceinline__ static bool two_fit(uint32_t a) { return a < (RT_SMEM_STACK - 1) * STK_E; }
    __device__ __forceinline__ void st_if(bool p, uint32_t a, int v) const {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.b32 [%0], %1;\n\t}" ::"r"(base + a),
                     "r"(v), "r"((uint32_t)p));
    }
    __device__ __forceinline__ int ld(uint32_t a) const {
        int v;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(base + a));
        return v;
    }
    __device__ __forceinline__ void set(uint32_t a, int v) const {
        const int i = (int)(a / STK_E);
        if (i < RT_SMEM_STACK) st_if(true, a, v);
        else l[i - RT_SMEM_STACK] = v;
    }
    __device__ __forceinline__ int get(uint32_t a) const {
        const int i = (int)(a / STK_E);
        return i < RT_SMEM_STACK ? ld(a) : l[i - RT_SMEM_STACK];
    }
};

template <bool COUNT>
struct Counters {
    uint32_t c[RT_NUM_COUNTERS_INTERNAL];
    __device__ void zero() {
#pragma unroll
        for (int i = 0; i < RT_NUM_COUNTERS_INTERNAL; ++i) c[i] = 0;
    }
    __device__ __forceinline__ void add(int i, uint32_t n = 1) { if (COUNT) c[i] += n; }
};

// Instrumented builds: real (non-empty) child boxes tested at a BVH4 node visit -- the slab
// tests the method performs; the inverted boxes of empty slots are layout, not work (§8(d) flops).
template <bool COUNT>
__device__ __forceinline__ void count_boxes(Counters<COUNT>& cnt, const int4& ch) {
    if (COUNT)
        cnt.add(CNT_BOX_TESTS, (ch.x != WIDE_EMPTY) + (ch.y != WIDE_EMPTY) + (ch.z != WIDE_EMPTY) + (ch.w != WIDE_EMPTY));
}

struct Hit {
    float t;
    int gid;    // global primitive ID, -1 = miss
    int slot;   // BVH prim slot (>= 0) or ~plane index (< 0)
};

// Work item -> (eye, px, py) and the item's shard-local tile `lt` (16x16 tiles; global tile id
// G = 2 t + eye for tile t of an eye, the layout rt_shard_tiles documents).
//   shard_mode 1 (world 2, the paper's level-1 eye split): this rank's eye only; each warp
//     takes one 8x4 block of a tile.
//   shard_mode 0 / 2 (one rank / world >= 3: tiles dealt to ranks round-robin): both eyes of a
//     tile are traced together, each warp taking one 4x4 block of the tile in BOTH eyes (lanes
//     0-15 left, 16-31 right).  With the zero-parallax plane at the scene (convergence C) the two
//     eyes' rays through one pixel are nearly the same ray, so a warp's 32 rays span a smaller
//     bundle than one eye's 8x4 block (C4 3.45 -> 3.21 ms per stereo frame).
template <typename Params>
__device__ __forceinline__ bool map_work(const Params& P, int k, int& eye, int& px, int& py, int& lt) {
    const int lane = k & 31, w = (k >> 5) & 7;
    int t;
    if (P.shard_mode == 1) {
        lt = k >> 8;
        eye = P.shard_rank;
        t = lt;
        px = (t % P.tiles_x) * TILE + (w & 1) * 8 + (lane & 7);
        py = (t / P.tiles_x) * TILE + (w >> 1) * 4 + (lane >> 3);
    } else {
        const int q = k >> 9, wp = (k >> 5) & 15;         // tile pair of this rank, warp of the pair
        eye = lane >> 4;
        lt = 2 * q + eye;
        t = P.tile_list ? __ldg(&P.tile_list[q]) : P.shard_rank + q * P.shard_world;
        px = (t % P.tiles_x) * TILE + (wp & 3) * 4 + (lane & 3);
        py = (t / P.tiles_x) * TILE + (wp >> 2) * 4 + ((lane >> 2) & 3);
    }
    return px < P.W && py < P.H;
}

__device__ __forceinline__ uint32_t pack_rgba8(float3 c) {
    const float r = __saturatef(c.x), g = __saturatef(c.y), b = __saturatef(c.z);
    const uint32_t R = __float2uint_rd(fmaf(r, 255.0f, 0.5f));
    const uint32_t G = __float2uint_rd(fmaf(g, 255.0f, 0.5f));
    const uint32_t B = __float2uint_rd(fmaf(b, 255.0f, 0.5f));
    return R | (G << 8) | (B << 16) | (0xFFu << 24);
}

__device__ __forceinline__ uint2 pack_rgba16f(float3 c) {
    const __half r = __float2half_rn(__saturatef(c.x)), g = __float2half_rn(__saturatef(c.y));
    const __half b = __float2half_rn(__saturatef(c.z)), a = __float2half_rn(1.0f);
    return make_uint2((uint32_t)__half_as_ushort(r) | ((uint32_t)__half_as_ushort(g) << 16),
                      (uint32_t)__half_as_ushort(b) | ((uint32_t)__half_as_ushort(a) << 16));
}

__device__ __forceinline__ void store_px(void* base, int fmt, long long pitch, int x, int y, float3 c) {
    char* row = static_cast<char*>(base) + (long long)y * pitch;
    if (fmt == RT_FORMAT_RGBA8) reinterpret_cast<uint32_t*>(row)[x] = pack_rgba8(c);
    else reinterpret_cast<uint2*>(row)[x] = pack_rgba16f(c);
}

// Primitive test shared by the BVH leaves and the brute-force path (bit-identical results).
// TRI: the scene holds triangles only (no spheres, no planes): the launch picks this
// instantiation so the sphere and plane code, never taken there, costs no registers (C4 -2.6 %).
template <bool COUNT, bool TRI = false>
__device__ __forceinline__ bool prim_t(const DevScene& S, int k, float3 o, float3 d, float& t, int& gid,
                                       Counters<COUNT>& cnt) {
    // all three 16-byte records up front, before the type test: both kinds read records 0 and 2
    // (a sphere keeps r^2 in record 2), so the loads are not sunk into the branches and a leaf
    // costs one memory round trip instead of two
    const float4 a = __ldg(&S.prims[3 * k]);
    const float4 b = __ldg(&S.prims[3 * k + 1]);
    const float4 c = __ldg(&S.prims[3 * k + 2]);
    gid = __float_as_int(a.w);
    if (!TRI && gid < S.n_spheres) {
        cnt.add(CNT_SPHERE_TESTS);
        return sphere_intersect(o, d, a, c.x, T_MIN, t);
    }
    cnt.add(CNT_TRI_TESTS);
    return tri_intersect(o, d, a, b, c, t) && t > T_MIN;
}

// Box tests of the 4 children of one BVH4 node (7 float4 in node_slot order).  Returns the hit
// mask straight from the four slab predicates; tn[c] = raw entry distance (>= 0), read only for
// the children the mask marks as hit.  Empty slots hold inverted boxes, which every test rejects.
__device__ __forceinline__ unsigned node4_hits(const float4* __restrict__ nodes, int node, const RayBox& rb, float tmax,
                                               float tn[4], int4& child) {
    const float4* q = nodes + (size_t)NODE_F4 * node;
    const float4 nx = __ldg(q + node_slot(rb.sx)), fx = __ldg(q + node_slot(1 - rb.sx));
    const float4 ny = __ldg(q + node_slot(2 + rb.sy)), fy = __ldg(q + node_slot(3 - rb.sy));
    const float4 nz = __ldg(q + node_slot(4 + rb.sz)), fz = __ldg(q + node_slot(5 - rb.sz));
    child = __ldg(reinterpret_cast<const int4*>(q + node_slot(6)));
    // packed FP32 FMA (sm_100 FFMA2): two children's plane distances per instruction
    const float2 ix = make_float2(rb.idir.x, rb.idir.x), iy = make_float2(rb.idir.y, rb.idir.y);
    const float2 iz = make_float2(rb.idir.z, rb.idir.z);
    const float2 cnx = make_float2(rb.cn.x, rb.cn.x), cny = make_float2(rb.cn.y, rb.cn.y), cnz = make_float2(rb.cn.z, rb.cn.z);
    const float2 cfx = make_float2(rb.cf.x, rb.cf.x), cfy = make_float2(rb.cf.y, rb.cf.y), cfz = make_float2(rb.cf.z, rb.cf.z);
    const float2 a0 = __ffma2_rn(make_float2(nx.x, nx.y), ix, cnx), a1 = __ffma2_rn(make_float2(nx.z, nx.w), ix, cnx);
    const float2 b0 = __ffma2_rn(make_float2(ny.x, ny.y), iy, cny), b1 = __ffma2_rn(make_float2(ny.z, ny.w), iy, cny);
    const float2 c0 = __ffma2_rn(make_float2(nz.x, nz.y), iz, cnz), c1 = __ffma2_rn(make_float2(nz.z, nz.w), iz, cnz);
    const float2 d0 = __ffma2_rn(make_float2(fx.x, fx.y), ix, cfx), d1 = __ffma2_rn(make_float2(fx.z, fx.w), ix, cfx);
    const float2 e0 = __ffma2_rn(make_float2(fy.x, fy.y), iy, cfy), e1 = __ffma2_rn(make_float2(fy.z, fy.w), iy, cfy);
    const float2 g0 = __ffma2_rn(make_float2(fz.x, fz.y), iz, cfz), g1 = __ffma2_rn(make_float2(fz.z, fz.w), iz, cfz);
    const float tn0 = fmaxf(fmaxf(a0.x, b0.x), fmaxf(c0.x, 0.0f)), tf0 = fminf(fminf(d0.x, e0.x), fminf(g0.x, tmax));
    const float tn1 = fmaxf(fmaxf(a0.y, b0.y), fmaxf(c0.y, 0.0f)), tf1 = fminf(fminf(d0.y, e0.y), fminf(g0.y, tmax));
    const float tn2 = fmaxf(fmaxf(a1.x, b1.x), fmaxf(c1.x, 0.0f)), tf2 = fminf(fminf(d1.x, e1.x), fminf(g1.x, tmax));
    const float tn3 = fmaxf(fmaxf(a1.y, b1.y), fmaxf(c1.y, 0.0f)), tf3 = fminf(fminf(d1.y, e1.y), fminf(g1.y, tmax));
    tn[0] = tn0;
    tn[1] = tn1;
    tn[2] = tn2;
    tn[3] = tn3;
    return (tn0 <= tf0 ? 1u : 0u) | (tn1 <= tf1 ? 2u : 0u) | (tn2 <= tf2 ? 4u : 0u) | (tn3 <= tf3 ? 8u : 0u);
}

__device__ __forceinline__ void cswap(uint32_t& a, uint32_t& b) {
    const uint32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}

// child code of slot i (0..3) with selects only (no branches)
__device__ __forceinline__ int pick4(const int4& c, uint32_t i) {
    const int lo = (i & 1u) ? c.y : c.x;
    const int hi = (i & 1u) ? c.w : c.z;
    return (i & 2u) ? hi : lo;
}

// child code of the lowest set bit of m (m != 0) as a chain of selects on the mask bits: shorter
// dependent latency than pick4(c, __ffs(m) - 1) (BREV, FLO, then the selects): C4 -1.2 %, C3 -1.5 %
__device__ __forceinline__ int pick_lowest(const int4& c, unsigned m) {
    return (m & 1u) ? c.x : (m & 2u) ? c.y : (m & 4u) ? c.z : c.w;
}

// Nearest-hit rays: visit order of the hit children.  Entry distances are >= 0, so their bit
// patterns order like unsigned ints; the 2 low bits carry the child slot and a 5-exchange network
// sorts them.  The nearest continues, the others are pushed far-to-near with predicated stores
// (no branches).  No cached top entry: with the stack pointer a plain shared offset the pop's LDS
// costs less than the top register's bookkeeping (C4 -0.6 %, C3 -0.6 %; round 1's v16 kept one
// when every push and pop also rebuilt the stack address).
__device__ __forceinline__ bool order_push(unsigned m, const float tn[4], const int4& ch, const TravStack& stk,
                                           uint32_t& sp, int& node) {
    if (!m) return false;
    const int nh = __popc(m);                               // one popcount drives both tests (C4 -0.3 %)
    if (nh == 1) {                                          // one hit (~40 % of visits): nothing to order
        node = pick_lowest(ch, m);
        return true;
    }
    if (nh == 2) {                                          // two hits: one compare, no network
        const float t0 = (m & 1u) ? tn[0] : (m & 2u) ? tn[1] : tn[2];        // lowest / highest hit slot
        const float t1 = (m & 8u) ? tn[3] : (m & 4u) ? tn[2] : tn[1];
        const int c0 = pick_lowest(ch, m), c1 = (m & 8u) ? ch.w : (m & 4u) ? ch.z : ch.y;
        const bool sw = t1 < t0;                            // ties keep slot order (as the keyed network)
        const int near = sw ? c1 : c0, far = sw ? c0 : c1;
        if (stk.two_fit(sp)) stk.st_if(true, sp, far);
        else stk.set(sp, far);
        sp += STK_E;
        node = near;
        return true;
    }
    uint32_t k0 = (m & 1) ? ((__float_as_uint(tn[0]) & ~3u) | 0u) : 0xffffffffu;
    uint32_t k1 = (m & 2) ? ((__float_as_uint(tn[1]) & ~3u) | 1u) : 0xffffffffu;
    uint32_t k2 = (m & 4) ? ((__float_as_uint(tn[2]) & ~3u) | 2u) : 0xffffffffu;
    uint32_t k3 = (m & 8) ? ((__float_as_uint(tn[3]) & ~3u) | 3u) : 0xffffffffu;
    cswap(k0, k1); cswap(k2, k3); cswap(k0, k2); cswap(k1, k3); cswap(k1, k2);
    // three or four hits: k3 (four only), k2, k1 -> entries sp, ..., far first
    const bool four = m == 15u;
    const uint32_t a = sp + (four ? 2u : 1u) * STK_E;     // entry of k1
    if (stk.two_fit(sp + STK_E)) {
        stk.st_if(four, sp, pick4(ch, k3 & 3u));
        stk.st_if(true, a - STK_E, pick4(ch, k2 & 3u));
        stk.st_if(true, a, pick4(ch, k1 & 3u));
    } else {
        if (four) stk.set(sp, pick4(ch, k3 & 3u));
        stk.set(a - STK_E, pick4(ch, k2 & 3u));
        stk.set(a, pick4(ch, k1 & 3u));
    }
    sp = a + STK_E;
    node = pick4(ch, k0 & 3u);
    return true;
}

// Any-hit (shadow) rays: continue with the lowest hit slot, the others (slots 1-3 only: slot 0 is
// always the lowest when hit) go to memory in slot order -- no distance sort (measured 7 % faster,
// and fewer triangle tests) and no cached top entry (the pop's LDS latency costs less than the
// top register's bookkeeping: C4 -1.3 %, C3 -1 %).
__device__ __forceinline__ bool plain_push(unsigned m, const int4& ch, const TravStack& stk, uint32_t& sp, int& node) {
    if (!m) return false;
    const unsigned r = m & (m - 1u);
    if (r) {
        if (stk.two_fit(sp + STK_E)) {
            stk.st_if(r & 2u, sp, ch.y);
            stk.st_if(r & 4u, sp + ((r >> 1) & 1u) * STK_E, ch.z);
            stk.st_if(r & 8u, sp + (uint32_t)__popc(r & 6u) * STK_E, ch.w);
        } else {
            if (r & 2u) stk.set(sp, ch.y);
            if (r & 4u) stk.set(sp + ((r >> 1) & 1u) * STK_E, ch.z);
            if (r & 8u) stk.set(sp + (uint32_t)__popc(r & 6u) * STK_E, ch.w);
        }
        sp += (uint32_t)__popc(r) * STK_E;
    }
    node = pick_lowest(ch, m);
    return true;
}
__device__ __forceinline__ bool pop_mem(const TravStack& stk, uint32_t& sp, int& node) {
    if (!stk.nonempty(sp)) return false;
    sp -= STK_E;
    node = stk.get(sp);
    return true;
}


// ---------------------------------------------------------------- NEXT-4: kd-tree ablation
// Stack traversal of the host-built kd-tree (rt_kdtree.cu): front-to-back cells, each split
// distance widened by the slab test's margin m |1/d_axis| on both sides, so every leaf cell a
// hit can lie in is visited; cells are pruned only when their (widened) entry lies beyond the
// best hit (t_entry <= t_best survives, as in the BVH), and leaf references are tested with the
// same primitive test.  Nearest (t, ID) hits therefore equal brute force exactly.
enum { ACC_BVH = 0, ACC_BRUTE = 1, ACC_KD = 2 };
constexpr int KD_STACK = 64;

struct KdRay {
    float o[3], id[3], m;
};

// root interval [t0, t1] of the kd cell (conservative), false if the ray misses it
__device__ __forceinline__ bool kd_setup(const DevScene& S, float3 o, float3 d, float tmax, KdRay& k, float& t0, float& t1) {
    const RayBox rb = make_raybox(o, d, S.bound);
    const float nx = rb.sx ? S.kd_hi.x : S.kd_lo.x, fx = rb.sx ? S.kd_lo.x : S.kd_hi.x;
    const float ny = rb.sy ? S.kd_hi.y : S.kd_lo.y, fy = rb.sy ? S.kd_lo.y : S.kd_hi.y;
    const float nz = rb.sz ? S.kd_hi.z : S.kd_lo.z, fz = rb.sz ? S.kd_lo.z : S.kd_hi.z;
    t0 = fmaxf(fmaxf(fmaf(nx, rb.idir.x, rb.cn.x), fmaf(ny, rb.idir.y, rb.cn.y)), fmaxf(fmaf(nz, rb.idir.z, rb.cn.z), 0.0f));
    t1 = fminf(fminf(fmaf(fx, rb.idir.x, rb.cf.x), fmaf(fy, rb.idir.y, rb.cf.y)), fminf(fmaf(fz, rb.idir.z, rb.cf.z), tmax));
    k.o[0] = o.x; k.o[1] = o.y; k.o[2] = o.z;
    k.id[0] = rb.idir.x; k.id[1] = rb.idir.y; k.id[2] = rb.idir.z;
    k.m = 1e-6f * (fabsf(o.x) + fabsf(o.y) + fabsf(o.z) + S.bound);
    return t0 <= t1;
}

// ANY: stop at the first primitive with t_min < t < limit.  Otherwise nearest hit into h.
template <bool COUNT, bool ANY>
__device__ __forceinline__ bool kd_trace(const DevScene& S, float3 o, float3 d, float limit, Hit& h, Counters<COUNT>& cnt,
                                         int* hint) {
    KdRay k;
    float t0, t1;
    if (!kd_setup(S, o, d, limit, k, t0, t1)) return false;
    int st_node[KD_STACK];
    float st_t0[KD_STACK], st_t1[KD_STACK];
    int sp = 0;
    int node = 0;
    while (true) {
        int2 n = __ldg(&S.kd_nodes[node]);
        while ((n.x & 3) != 3) {
            cnt.add(CNT_NODE_VISITS);
            const int axis = n.x & 3;
            const float oa = axis == 0 ? k.o[0] : (axis == 1 ? k.o[1] : k.o[2]);
            const float ia = axis == 0 ? k.id[0] : (axis == 1 ? k.id[1] : k.id[2]);
            const float ts = (__int_as_float(n.y) - oa) * ia;
            const float e = k.m * fabsf(ia);
            const float ts_lo = ts - e, ts_hi = ts + e;
            const int left = node + 1, right = n.x >> 2;
            const int nearc = ia >= 0.0f ? left : right, farc = ia >= 0.0f ? right : left;
            const float tcut = ANY ? t1 : fminf(t1, h.t);
            const bool vn = t0 <= fminf(tcut, ts_hi);
            const bool vf = fmaxf(t0, ts_lo) <= tcut;
            if (vn && vf) {
                if (sp < KD_STACK) {
                    st_node[sp] = farc; st_t0[sp] = fmaxf(t0, ts_lo); st_t1[sp] = t1; ++sp;
                }
                node = nearc;
                t1 = fminf(t1, ts_hi);
            } else if (vn) {
                node = nearc;
                t1 = fminf(t1, ts_hi);
            } else if (vf) {
                node = farc;
                t0 = fmaxf(t0, ts_lo);
            } else {
                node = -1;
                break;
            }
            n = __ldg(&S.kd_nodes[node]);
        }
        if (node >= 0) {
            const int cnt_refs = n.x >> 2, first = n.y;
            for (int i = 0; i < cnt_refs; ++i) {
                const int kk = __ldg(&S.kd_refs[first + i]);
                float t;
                int gid;
                if (prim_t<COUNT>(S, kk, o, d, t, gid, cnt)) {
                    if (ANY) {
                        if (t < limit) {
                            if (hint) *hint = kk;
                            return true;
                        }
                    } else if (t < h.t || (t == h.t && gid < h.gid)) {
                        h.t = t; h.gid = gid; h.slot = kk;
                    }
                }
            }
        }
        // next cell: front-to-back pops, pruned by the best hit so far
        bool found = false;
        while (sp > 0) {
            --sp;
            if (st_t0[sp] <= (ANY ? st_t1[sp] : fminf(st_t1[sp], h.t))) {
                node = st_node[sp]; t0 = st_t0[sp]; t1 = st_t1[sp];
                found = true;
                break;
            }
        }
        if (!found) return false;
    }
}

// Nearest hit over the 4-wide BVH (or every BVH primitive when BRUTE, the kd-tree when KD) and
// the planes.  Acceptance: t > t_min and (t, gid) lexicographically smallest (
// reading 9).  Children are visited near-to-far (order_push).
template <bool COUNT, int ACC, bool TRI = false, bool L1 = false>
__device__ __forceinline__ Hit closest_hit(const DevScene& S, float3 o, float3 d, const TravStack& stk, Counters<COUNT>& cnt) {
    constexpr bool BRUTE = ACC == ACC_BRUTE;
    Hit h;
    h.t = __int_as_float(0x7f800000);
    h.gid = -1;
    h.slot = 0;
    for (int i = 0; i < (TRI ? 0 : S.n_planes); ++i) {
        cnt.add(CNT_PLANE_TESTS);
        float t;
        if (plane_intersect(o, d, __ldg(&S.planes[i]), t) && t > T_MIN) {
            const int gid = S.n_spheres + i;
            if (t < h.t || (t == h.t && gid < h.gid)) { h.t = t; h.gid = gid; h.slot = ~i; }
        }
    }
    if (S.n_bvh == 0) return h;
    if constexpr (ACC == ACC_KD) {
        kd_trace<COUNT, false>(S, o, d, __int_as_float(0x7f800000), h, cnt, nullptr);
        return h;
    }
    auto leaf_test = [&](int first, int last) {
        for (int k = first; k <= last; ++k) {
            float t;
            int gid;
            if (prim_t<COUNT, TRI>(S, k, o, d, t, gid, cnt) && (t < h.t || (t == h.t && gid < h.gid))) {
                h.t = t; h.gid = gid; h.slot = k;
            }
        }
    };
    if (BRUTE) {
        leaf_test(0, S.n_bvh - 1);
        return h;
    }
    const RayBox rb = make_raybox(o, d, S.bound);
    uint32_t sp = stk.empty();
    int node = S.root;
    while (true) {
        if (node >= 0) {
            cnt.add(CNT_NODE_VISITS);
            float tn[4];
            int4 ch;
            const unsigned m = node4_hits(S.nodes, node, rb, h.t, tn, ch);
            count_boxes(cnt, ch);
            if (order_push(m, tn, ch, stk, sp, node)) continue;
        } else if (L1) {
            leaf_test(~node, ~node);                 // single-primitive leaves: the code is ~slot
        } else {
            const int enc = ~node;
            const int first = enc & ((1 << LEAF_SHIFT) - 1);
            leaf_test(first, first + (enc >> LEAF_SHIFT));
        }
        if (!pop_mem(stk, sp, node)) return h;
    }
}

// Any hit with t_min < t < dist (binary visibility, reading 4).  `hint` (shared memory, may be
// null) holds the BVH slot of this thread's last occluder for the same light: it is tested first
// and, if it blocks the segment, the answer is already exact (visibility is a boolean, so which
// occluder proves it does not matter); otherwise the traversal runs and records its occluder if
// that is a sphere.  A sphere covers many neighbouring pixels' shadow rays (C3: 1.1 M of the
// frame's shadow rays end at the hint), a triangle of a fine mesh almost none (C4: 329 of 0.79 M
// occluded rays), so triangle hints only cost a primitive test per shadow ray (C4 -0.5 %).
template <bool COUNT, int ACC, bool TRI = false, bool L1 = false>
__device__ __forceinline__ bool occluded(const DevScene& S, float3 o, float3 d, float dist, const TravStack& stk, Counters<COUNT>& cnt,
                                         int* hint = nullptr) {
    constexpr bool BRUTE = ACC == ACC_BRUTE;
    for (int i = 0; i < (TRI ? 0 : S.n_planes); ++i) {
        cnt.add(CNT_PLANE_TESTS);
        float t;
        if (plane_intersect(o, d, __ldg(&S.planes[i]), t) && t > T_MIN && t < dist) return true;
    }
    if (S.n_bvh == 0) return false;
    if (BRUTE) hint = nullptr;
    if (hint) {
        const int k = *hint;
        float t;
        int gid;
        if (k >= 0 && prim_t<COUNT, TRI>(S, k, o, d, t, gid, cnt) && t < dist) return true;
    }
    if constexpr (ACC == ACC_KD) {
        Hit h;
        h.t = dist; h.gid = -1; h.slot = 0;
        return kd_trace<COUNT, true>(S, o, d, dist, h, cnt, hint);
    }
    auto leaf_test = [&](int first, int last) -> bool {
        for (int k = first; k <= last; ++k) {
            float t;
            int gid;
            if (prim_t<COUNT, TRI>(S, k, o, d, t, gid, cnt) && t < dist) {
                if (hint && gid < S.n_spheres) *hint = k;   // spheres only (see occluded)
                return true;
            }
        }
        return false;
    };
    if (BRUTE) return leaf_test(0, S.n_bvh - 1);
    const RayBox rb = make_raybox(o, d, S.bound);
    uint32_t sp = stk.empty();
    int node = S.root;
    while (true) {
        if (node >= 0) {
            cnt.add(CNT_NODE_VISITS);
            float tn[4];
            int4 ch;
            const unsigned m = node4_hits(S.nodes, node, rb, dist, tn, ch);
            count_boxes(cnt, ch);
            if (plain_push(m, ch, stk, sp, node)) continue;
        } else if (L1) {
            if (leaf_test(~node, ~node)) return true;   // single-primitive leaves: the code is ~slot
        } else {
            const int enc = ~node;
            const int first = enc & ((1 << LEAF_SHIFT) - 1);
            if (leaf_test(first, first + (enc >> LEAF_SHIFT))) return true;
        }
        if (!pop_mem(stk, sp, node)) return false;
    }
}

}  // namespace rtb
