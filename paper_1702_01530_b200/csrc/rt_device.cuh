// rt_device.cuh -- device-side data layout and FP32 intersectors of the B200 stereo ray tracer.
//
// Layout in HBM:
//   nodes  : BVH4 nodes, 7 x float4 = 112 B each, stored in slot order
//              lo.x[4] hi.x[4] lo.y[4] child[4] hi.y[4] lo.z[4] hi.z[4]   (node_slot below)
//            child >= 0 internal node, WIDE_EMPTY unused slot (inverted box), child < 0 leaf:
//            ~child = (count-1) << 24 | first_prim.
//            (Measured and rejected layouts -- 8-wide, binary16-compressed, 128-B padded nodes --
//            are in git history before the round-2 pruning.)
//   prims  : 3 x float4 = 48 B per BVH primitive, in leaf (Morton) order
//              triangle: (v0.xyz, gid) (e1.xyz, mat) (e2.xyz, 0)        -- SPEC:170 Moller-Trumbore
//              sphere  : (c.xyz,  gid) (r, r^2, 0, mat) (r^2, 0, 0, 0)
//            gid < n_spheres <=> sphere (global IDs: spheres, planes, triangles).
//   planes : (n^.xyz, k) float4 + mat int, tested linearly (infinite, not in the BVH)
//   mats   : 3 x float4: (kd.xyz, shininess) (ks.xyz, kr) (kt, ior, 0, 0)
//   lights : 2 x float4: (pos.xyz, 0) (I.xyz, 0)
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace rtb {

constexpr float T_MIN = 1e-4f;     // SPEC.md:156 t_min
constexpr float BIAS = 1e-4f;      // SPEC.md:156 shadow_bias (also reflection/refraction origins)
constexpr int MAX_DEPTH = 16;
constexpr int BVH_W = 4;                               // children per node
constexpr int NODE_DATA_F4 = 7;                        // float4 per node: lo/hi x,y,z + child codes
constexpr int NODE_F4 = NODE_DATA_F4;                  // node stride in float4
constexpr int STACK_CAP = (BVH_W - 1) * 64 + 2;       // traversal stack: W-1 siblings per level, depth <= 64
// Storage slot (16-byte unit) of array a = 0 lo.x, 1 hi.x, 2 lo.y, 3 hi.y, 4 lo.z, 5 hi.z,
// 6 child codes.  The child codes sit in slot 3, between lo.y and hi.y.  A 112-byte
// node starts on a 32-byte sector boundary or 16 bytes past one; either way the codes then share
// their sector with lo.y or hi.y -- both always loaded (the near and far y planes) -- so the codes'
// load, which ptxas issues only after the box tests, hits a sector already on its way to L1
// instead of costing a second L2 round trip.
__host__ __device__ constexpr int node_slot(int a) {
    return a == 6 ? 3 : (a >= 3 ? a + 1 : a);
}
constexpr int LEAF_SHIFT = 24;     // leaf encoding: ~((count-1) << 24 | first)
constexpr int TILE = 16;
constexpr int WIDE_EMPTY = 0x7fffffff;   // unused BVH4 child slot
constexpr int TRAV_DONE = (int)0x80000000;  // traversal finished (not a valid leaf code)

// ------------------------------------------------------------------ node codec (build / refit)
// Writes one node from its children's boxes and codes (code == WIDE_EMPTY: unused slot).
__device__ inline void node_write(float4* q, const float3* lo, const float3* hi, const int* code) {
    float* o = reinterpret_cast<float*>(q);
    int* oc = reinterpret_cast<int*>(o) + node_slot(6) * BVH_W;
    for (int c = 0; c < BVH_W; ++c) {
        if (code[c] == WIDE_EMPTY) {
            // inverted box (lo = +1e30, hi = -1e30): every slab test rejects it, so the
            // traversal needs no per-slot validity test
            for (int k = 0; k < 3; ++k) {
                o[node_slot(2 * k) * BVH_W + c] = 1e30f;
                o[node_slot(2 * k + 1) * BVH_W + c] = -1e30f;
            }
        } else {
            o[node_slot(0) * BVH_W + c] = lo[c].x; o[node_slot(1) * BVH_W + c] = hi[c].x;
            o[node_slot(2) * BVH_W + c] = lo[c].y; o[node_slot(3) * BVH_W + c] = hi[c].y;
            o[node_slot(4) * BVH_W + c] = lo[c].z; o[node_slot(5) * BVH_W + c] = hi[c].z;
        }
        oc[c] = code[c];
    }
}

__device__ inline int node_code(const float4* q, int c) {
    return reinterpret_cast<const int*>(q)[node_slot(6) * BVH_W + c];
}

// Box of child c as stored (decoded outward-rounded for compressed nodes; empty = inverted).
__device__ inline void node_child_box(const float4* q, int c, float3& lo, float3& hi) {
    const float* r = reinterpret_cast<const float*>(q);
    lo = make_float3(r[node_slot(0) * BVH_W + c], r[node_slot(2) * BVH_W + c], r[node_slot(4) * BVH_W + c]);
    hi = make_float3(r[node_slot(1) * BVH_W + c], r[node_slot(3) * BVH_W + c], r[node_slot(5) * BVH_W + c]);
}

struct DevScene {
    const float4* __restrict__ nodes;
    const float4* __restrict__ prims;
    const float4* __restrict__ planes;
    const int* __restrict__ plane_mat;
    const float4* __restrict__ mats;
    const float4* __restrict__ lights;
    int n_bvh;          // primitives in the BVH
    int root;           // >= 0 internal node, < 0 leaf encoding, meaningless if n_bvh == 0
    int n_spheres;
    int n_planes;
    int n_lights;
    int refractive;     // some material has kt > 0 (else the launch may pick the opaque instantiation)
    float bound;        // max |x|+|y|+|z| over the BVH bounds (box-test margin scale)
    float3 ambient;
    float3 background;
    // NEXT-4 ablation: kd-tree over the same primitive records (null unless rt_kdtree_build ran)
    const int2* __restrict__ kd_nodes;
    const int* __restrict__ kd_refs;
    float3 kd_lo, kd_hi;
};

struct DevCamera {
    float3 eye[2];
    float3 f, r, u;
    float tha, th;      // tan(vfov/2) * aspect, tan(vfov/2)
    float sigma[2];     // off-axis shift per eye
};

// ------------------------------------------------------------------ float3 helpers
__device__ __forceinline__ float3 f3(float x, float y, float z) { return make_float3(x, y, z); }
__device__ __forceinline__ float3 xyz(float4 a) { return make_float3(a.x, a.y, a.z); }
__device__ __forceinline__ float3 operator+(float3 a, float3 b) { return f3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ float3 operator-(float3 a, float3 b) { return f3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ float3 operator*(float3 a, float s) { return f3(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ float3 operator*(float3 a, float3 b) { return f3(a.x * b.x, a.y * b.y, a.z * b.z); }
__device__ __forceinline__ float dot(float3 a, float3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ float3 cross(float3 a, float3 b) {
    return f3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ float3 normalize(float3 a) { return a * rsqrtf(dot(a, a)); }
// sqrt and reciprocal through the MUFU approximations (~2 ulp), like normalize above: the IEEE
// versions carry a slow-path call whose register saves spill the traversal state around them
__device__ __forceinline__ float fsqrt(float x) { return x > 0.0f ? x * rsqrtf(x) : 0.0f; }
__device__ __forceinline__ float frcp(float x) { return __fdividef(1.0f, x); }
__device__ __forceinline__ float sqrt_sph(float x) { return fsqrt(x); }     // sphere test
__device__ __forceinline__ float sqrt_dist(float x) { return fsqrt(x); }    // shadow-ray length, refraction
__device__ __forceinline__ float rcp_dist(float x) { return frcp(x); }
// 1/d of the ray setup: the compiler's reciprocal (MUFU under --use_fast_math); an explicit
// __fdividef here measured C2 -5 % but C4 and C3 +4 % (DESIGN.md §5 v19)
__device__ __forceinline__ float rcp_inv(float x) { return 1.0f / x; }
__device__ __forceinline__ float3 fma3(float3 a, float s, float3 b) {
    return f3(fmaf(a.x, s, b.x), fmaf(a.y, s, b.y), fmaf(a.z, s, b.z));
}

// ------------------------------------------------------------------ intersectors (FP32)
// Moller-Trumbore with stored v0, e1, e2: inclusive edges, det == 0 -> miss.
// Division-free acceptance: the barycentric numerators are compared against |det| after a
// sign flip, and t = t_num / det is formed only for accepted hits.  Returns the raw t (the
// caller applies t_min / t_best).
__device__ __forceinline__ bool tri_intersect(float3 o, float3 d, float4 a, float4 b, float4 c, float& t) {
    const float3 e1 = xyz(b), e2 = xyz(c);
    const float3 p = cross(d, e2);
    const float det_s = dot(e1, p);
    const uint32_t sgn = __float_as_uint(det_s) & 0x80000000u;
    const float det = fabsf(det_s);
    const float3 s = o - xyz(a);
    const float u = __uint_as_float(__float_as_uint(dot(s, p)) ^ sgn);
    if (!(det > 0.0f) || u < 0.0f || u > det) return false;
    const float3 q = cross(s, e1);
    const float v = __uint_as_float(__float_as_uint(dot(d, q)) ^ sgn);
    if (v < 0.0f || u + v > det) return false;
    t = __fdividef(__uint_as_float(__float_as_uint(dot(e2, q)) ^ sgn), det);
    return true;
}

// Sphere |o + t d - c| = r, |d| = 1, numerically stable form (reading 21):
// disc = r^2 - |oc - (oc.d) d|^2, roots -b -/+ sqrt(disc); returns the smallest root > tmin.
__device__ __forceinline__ bool sphere_intersect(float3 o, float3 d, float4 a, float r2, float tmin, float& t) {
    const float3 oc = o - xyz(a);
    const float bb = dot(oc, d);
    const float3 f = oc - d * bb;
    const float disc = r2 - dot(f, f);
    if (disc < 0.0f) return false;
    const float q = sqrt_sph(disc);
    const float cc = dot(oc, oc) - r2;
    const float h = bb > 0.0f ? -(bb + q) : (q - bb);     // larger-magnitude root
    float t0, t1;
    if (h != 0.0f) { t0 = __fdividef(cc, h); t1 = h; } else { t0 = 0.0f; t1 = 0.0f; }
    if (t0 > t1) { const float x = t0; t0 = t1; t1 = x; }
    if (t0 > tmin) { t = t0; return true; }
    if (t1 > tmin) { t = t1; return true; }
    return false;
}

// Plane n^.x = k: t = (k - n^.o) / (n^.d); n^.d == 0 -> miss.
__device__ __forceinline__ bool plane_intersect(float3 o, float3 d, float4 p, float& t) {
    const float3 n = xyz(p);
    const float den = dot(n, d);
    if (den == 0.0f) return false;
    t = __fdividef(p.w - dot(n, o), den);   // like the sphere and triangle tests: no IEEE-division slow-path call (and the spills around it)
    return true;
}

// Conservative slab-test setup.  Each box plane is tested as fma(plane, 1/d, c) with per-ray
// constants c = -(o -/+ m)/d chosen so that entry distances are rounded down and exit
// distances up by m = 1e-6 (|o|_1 + B) world units -- far above the FP32 error of every
// primitive test -- so the BVH never culls a primitive the brute-force loop would accept
// (GPU LBVH == GPU brute force, bit-exact).  The near/far plane of each axis is
// picked once per ray from the direction's sign (no per-box min/max of slab pairs).
struct RayBox {
    float3 idir;
    float3 cn;    // near-plane constants
    float3 cf;    // far-plane constants
    int sx, sy, sz;   // 1 if d < 0 on that axis (near plane = hi)
};

__device__ __forceinline__ float safe_inv(float x) {
    const float ax = fabsf(x);
    // approximate (1 ulp) reciprocal: the slab margin m covers 8x its effect on t
    return rcp_inv(ax < 1e-30f ? copysignf(1e-30f, x) : x);
}

__device__ __forceinline__ RayBox make_raybox(float3 o, float3 d, float bound) {
    RayBox rb;
    const float m = 1e-6f * (fabsf(o.x) + fabsf(o.y) + fabsf(o.z) + bound);
    rb.idir = f3(safe_inv(d.x), safe_inv(d.y), safe_inv(d.z));
    const float3 clo = f3(-(o.x + m) * rb.idir.x, -(o.y + m) * rb.idir.y, -(o.z + m) * rb.idir.z);
    const float3 chi = f3(-(o.x - m) * rb.idir.x, -(o.y - m) * rb.idir.y, -(o.z - m) * rb.idir.z);
    rb.sx = rb.idir.x < 0.0f;
    rb.sy = rb.idir.y < 0.0f;
    rb.sz = rb.idir.z < 0.0f;
    rb.cn = f3(rb.sx ? chi.x : clo.x, rb.sy ? chi.y : clo.y, rb.sz ? chi.z : clo.z);
    rb.cf = f3(rb.sx ? clo.x : chi.x, rb.sy ? clo.y : chi.y, rb.sz ? clo.z : chi.z);
    return rb;
}

}  // namespace rtb
