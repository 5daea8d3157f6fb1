// Host binned-SAH BVH2 over the leaf-order primitive boxes: an experiment (env RT_HOST_SAH=1)
// that measures how much traversal the device LBVH + treelet build leaves on the table.  It
// replaces the BVH2 topology and boxes (left / right / node_lo / node_hi; leaves are the same
// sorted primitive slots) before the device BVH2 -> BVH4 collapse, so everything downstream is
// the product path.  SURVEY.md §8(f) NEXT-4; DESIGN.md §5.
#include <algorithm>
#include <cfloat>
#include <vector>

#include "rt_internal.h"

namespace rtb {
namespace {
struct Box {
    float lo[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, hi[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    void grow(const Box& b) {
        for (int a = 0; a < 3; ++a) { lo[a] = std::min(lo[a], b.lo[a]); hi[a] = std::max(hi[a], b.hi[a]); }
    }
    float area() const {
        if (lo[0] > hi[0]) return 0.0f;
        const float x = hi[0] - lo[0], y = hi[1] - lo[1], z = hi[2] - lo[2];
        return x * y + y * z + z * x;
    }
};
constexpr int BINS = 32;
}  // namespace

void sah_build_host(const float4* leaf_lo, const float4* leaf_hi, int n, int* left, int* right, float4* node_lo,
                    float4* node_hi) {
    std::vector<Box> box(n);
    std::vector<float> cen(3 * (size_t)n);
    for (int i = 0; i < n; ++i) {
        const float l[3] = {leaf_lo[i].x, leaf_lo[i].y, leaf_lo[i].z}, h[3] = {leaf_hi[i].x, leaf_hi[i].y, leaf_hi[i].z};
        for (int a = 0; a < 3; ++a) {
            box[i].lo[a] = l[a];
            box[i].hi[a] = h[a];
            cen[3 * (size_t)i + a] = 0.5f * (l[a] + h[a]);
        }
    }
    std::vector<int> idx(n);
    for (int i = 0; i < n; ++i) idx[i] = i;
    struct Task { int begin, end, node; };
    std::vector<Task> stack{{0, n, 0}};
    int next_node = 1;
    auto emit = [&](int b, int e) -> int {           // child code: ~slot or a new internal node
        if (e - b == 1) return ~idx[b];
        const int id = next_node++;
        stack.push_back({b, e, id});
        return id;
    };
    while (!stack.empty()) {
        const Task t = stack.back();
        stack.pop_back();
        Box nb, cb;
        for (int i = t.begin; i < t.end; ++i) {
            nb.grow(box[idx[i]]);
            Box c;
            for (int a = 0; a < 3; ++a) c.lo[a] = c.hi[a] = cen[3 * (size_t)idx[i] + a];
            cb.grow(c);
        }
        node_lo[t.node] = make_float4(nb.lo[0], nb.lo[1], nb.lo[2], 0.0f);
        node_hi[t.node] = make_float4(nb.hi[0], nb.hi[1], nb.hi[2], 0.0f);
        int best_axis = -1, best_bin = 0;
        float best_cost = FLT_MAX;
        for (int a = 0; a < 3; ++a) {
            const float ext = cb.hi[a] - cb.lo[a];
            if (!(ext > 0.0f)) continue;
            Box bb[BINS];
            int bc[BINS] = {0};
            const float k = BINS * (1.0f - 1e-6f) / ext;
            for (int i = t.begin; i < t.end; ++i) {
                const int b = std::min(BINS - 1, (int)((cen[3 * (size_t)idx[i] + a] - cb.lo[a]) * k));
                bb[b].grow(box[idx[i]]);
                ++bc[b];
            }
            float ra[BINS];
            int rc[BINS];
            Box acc;
            int cnt = 0;
            for (int b = BINS - 1; b > 0; --b) {
                acc.grow(bb[b]);
                cnt += bc[b];
                ra[b] = acc.area();
                rc[b] = cnt;
            }
            acc = Box();
            cnt = 0;
            for (int b = 0; b < BINS - 1; ++b) {
                acc.grow(bb[b]);
                cnt += bc[b];
                if (cnt == 0 || rc[b + 1] == 0) continue;
                const float c = acc.area() * cnt + ra[b + 1] * rc[b + 1];
                if (c < best_cost) { best_cost = c; best_axis = a; best_bin = b; }
            }
        }
        int mid;
        if (best_axis < 0) {
            mid = (t.begin + t.end) / 2;                 // coincident centroids: split the list
        } else {
            const float ext = cb.hi[best_axis] - cb.lo[best_axis];
            const float k = BINS * (1.0f - 1e-6f) / ext;
            const int a = best_axis;
            int* p = std::partition(idx.data() + t.begin, idx.data() + t.end, [&](int s) {
                return std::min(BINS - 1, (int)((cen[3 * (size_t)s + a] - cb.lo[a]) * k)) <= best_bin;
            });
            mid = (int)(p - idx.data());
            if (mid == t.begin || mid == t.end) mid = (t.begin + t.end) / 2;
        }
        left[t.node] = emit(t.begin, mid);
        right[t.node] = emit(mid, t.end);
    }
}
}  // namespace rtb
