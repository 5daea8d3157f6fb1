// rt_kdtree.cu -- NEXT-4 ablation (Table 1 "Kd-trees: binary
// search for the primitive intersected by the ray, simple traversal, little memory / time-
// consuming construction with SAH split search, greater depth than the BVH").
//
// A binned-SAH kd-tree over the BVH's primitive records, built on the HOST from a copy of them
// (the product path builds and traverses the device LBVH; this structure exists only to measure
// Table 1's comparison on the same scenes and the same FP32 intersectors).  Primitives whose
// AABB straddles a split plane are referenced in both children (closed intervals), so every
// primitive is covered by the union of the leaf cells that reference it; the device traversal
// (rt_trace.cuh, kd_*) widens every split distance by the same conservative margin as the BVH
// slab test, so it visits every leaf cell a hit can lie in and the nearest (t, ID) hit equals
// brute force exactly.
//
// Node encoding (int2, preorder, left child = node + 1):
//   inner: x = axis | (right child index << 2), y = split position (float bits)
//   leaf:  x = 3 | (reference count << 2),      y = first reference
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "rt_internal.h"

namespace {

constexpr int KD_BINS = 32;
constexpr double KD_COST_TRAV = 1.0;     // SAH: one traversal step
constexpr double KD_COST_ISECT = 1.5;    // SAH: one primitive test
constexpr double KD_EMPTY_BONUS = 0.8;   // cost factor for splits that cut off empty space

struct Builder {
    const float* box;    // 6 per primitive: lo xyz, hi xyz
    int max_leaf, max_depth;
    std::vector<int2> nodes;
    std::vector<int> refs;
    int depth = 0, leaves = 0;

    static double area(const double lo[3], const double hi[3]) {
        const double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
        return 2.0 * (dx * dy + dy * dz + dz * dx);
    }

    void leaf(const std::vector<int>& r, int d) {
        int2 n;
        n.x = 3 | ((int)r.size() << 2);
        n.y = (int)refs.size();
        refs.insert(refs.end(), r.begin(), r.end());
        nodes.push_back(n);
        ++leaves;
        depth = std::max(depth, d);
    }

    // SAH split search over KD_BINS bins per axis; returns false if a leaf is cheaper
    bool find_split(const std::vector<int>& r, const double lo[3], const double hi[3], int& axis, float& split) const {
        const double N = (double)r.size();
        const double sa = area(lo, hi);
        double best = KD_COST_ISECT * N;                  // leaf cost
        bool found = false;
        for (int a = 0; a < 3; ++a) {
            const double ext = hi[a] - lo[a];
            if (!(ext > 0.0)) continue;
            int cs[KD_BINS] = {0}, ce[KD_BINS] = {0};      // primitives starting / ending in bin
            for (int k : r) {
                const double s = box[6 * k + a], e = box[6 * k + 3 + a];
                int bs = (int)((s - lo[a]) / ext * KD_BINS), be = (int)((e - lo[a]) / ext * KD_BINS);
                bs = std::min(std::max(bs, 0), KD_BINS - 1);
                be = std::min(std::max(be, 0), KD_BINS - 1);
                ++cs[bs];
                ++ce[be];
            }
            // plane j (between bins j-1 and j): left = primitives starting in bins < j,
            // right = primitives ending in bins >= j
            int nl = 0, nr = (int)r.size();
            for (int j = 1; j < KD_BINS; ++j) {
                nl += cs[j - 1];
                nr -= ce[j - 1];
                const double p = lo[a] + ext * j / KD_BINS;
                double llo[3] = {lo[0], lo[1], lo[2]}, lhi[3] = {hi[0], hi[1], hi[2]};
                double rlo[3] = {lo[0], lo[1], lo[2]}, rhi[3] = {hi[0], hi[1], hi[2]};
                lhi[a] = p;
                rlo[a] = p;
                double c = KD_COST_TRAV + KD_COST_ISECT * (area(llo, lhi) * nl + area(rlo, rhi) * nr) / sa;
                if (nl == 0 || nr == 0) c *= KD_EMPTY_BONUS;
                if (c < best) {
                    best = c;
                    axis = a;
                    split = (float)p;
                    found = true;
                }
            }
        }
        return found;
    }

    void build(std::vector<int>& r, const double lo[3], const double hi[3], int d) {
        int axis = 0;
        float split = 0.0f;
        if ((int)r.size() <= max_leaf || d >= max_depth || !find_split(r, lo, hi, axis, split)) {
            leaf(r, d);
            return;
        }
        std::vector<int> L, R;
        L.reserve(r.size() / 2 + 1);
        R.reserve(r.size() / 2 + 1);
        for (int k : r) {                                 // closed intervals: straddlers go both ways
            if (box[6 * k + axis] <= split) L.push_back(k);
            if (box[6 * k + 3 + axis] >= split) R.push_back(k);
        }
        if (L.size() == r.size() && R.size() == r.size()) {   // the plane cut nothing off
            leaf(r, d);
            return;
        }
        std::vector<int>().swap(r);
        const size_t me = nodes.size();
        nodes.push_back(make_int2(0, 0));
        double llo[3] = {lo[0], lo[1], lo[2]}, lhi[3] = {hi[0], hi[1], hi[2]};
        double rlo[3] = {lo[0], lo[1], lo[2]}, rhi[3] = {hi[0], hi[1], hi[2]};
        lhi[axis] = split;
        rlo[axis] = split;
        build(L, llo, lhi, d + 1);
        const int right = (int)nodes.size();
        build(R, rlo, rhi, d + 1);
        int sb;
        memcpy(&sb, &split, 4);
        nodes[me] = make_int2(axis | (right << 2), sb);
    }
};

}  // namespace

namespace rtb {

// AABBs of the device primitive records (leaf order; 3 float4 each, rt_device.cuh), rounded
// outward; then the kd-tree over them.
void kd_build_host(const float4* prims, int n, int n_spheres, int max_leaf, int max_depth, KdHost& out) {
    std::vector<float> box(6 * (size_t)n);
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int k = 0; k < n; ++k) {
        const float4 a = prims[3 * k], b = prims[3 * k + 1], c = prims[3 * k + 2];
        int gid;
        memcpy(&gid, &a.w, 4);
        double l[3], h[3];
        if (gid < n_spheres) {
            const double cc[3] = {a.x, a.y, a.z};
            for (int i = 0; i < 3; ++i) { l[i] = cc[i] - b.x; h[i] = cc[i] + b.x; }
        } else {
            const double v0[3] = {a.x, a.y, a.z}, e1[3] = {b.x, b.y, b.z}, e2[3] = {c.x, c.y, c.z};
            for (int i = 0; i < 3; ++i) {
                l[i] = std::min(v0[i], std::min(v0[i] + e1[i], v0[i] + e2[i]));
                h[i] = std::max(v0[i], std::max(v0[i] + e1[i], v0[i] + e2[i]));
            }
        }
        for (int i = 0; i < 3; ++i) {
            float fl = (float)l[i], fh = (float)h[i];
            if ((double)fl > l[i]) fl = nextafterf(fl, -INFINITY);
            if ((double)fh < h[i]) fh = nextafterf(fh, INFINITY);
            box[6 * (size_t)k + i] = fl;
            box[6 * (size_t)k + 3 + i] = fh;
            lo[i] = std::min(lo[i], (double)fl);
            hi[i] = std::max(hi[i], (double)fh);
        }
    }
    Builder B;
    B.box = box.data();
    B.max_leaf = std::max(max_leaf, 1);
    B.max_depth = max_depth > 0 ? max_depth : (int)std::lround(8.0 + 1.3 * std::log2((double)std::max(n, 1)));
    std::vector<int> all(n);
    for (int k = 0; k < n; ++k) all[k] = k;
    B.nodes.reserve(4 * (size_t)n / std::max(B.max_leaf, 1) + 16);
    B.refs.reserve(2 * (size_t)n + 16);
    if (n > 0) B.build(all, lo, hi, 0);
    out.nodes.swap(B.nodes);
    out.refs.swap(B.refs);
    out.depth = B.depth;
    out.leaves = B.leaves;
    for (int i = 0; i < 3; ++i) {
        out.lo[i] = (float)lo[i];
        out.hi[i] = (float)hi[i];
    }
}

}  // namespace rtb
