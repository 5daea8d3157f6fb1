// rt_wave.cu -- the hot path as a bounce-level wavefront.
//
// The paper synthesises each stereo channel by tracing every pixel (§3 Fig. 2);
// here both channels' pixels form one work list (level 1 and level 2 parallelism fused) and the
// Whitted ray tree (S:190-208 + refraction) is evaluated breadth-first, one bounce level at a
// time, so every kernel runs ONE kind of ray in dense, spatially ordered batches:
//
//   level L:  k_extend   nearest hit of every tree ray of the level (L = 0: primary rays are
//                        generated in registers from the work item)
//             k_shade    hit point, facing normal, ambient*kd; for each light with n.l > 0 the
//                        Phong term w*(kd*I*ndl + ks*I*spec) is computed and a shadow ray is
//                        appended to that light's queue; reflection/refraction children (with
//                        their path weights) go to the next level's queue; misses add w*bg
//             k_occlude  any hit of every shadow ray; unoccluded rays add their term
//   then      k_finalize clamps and packs RGBA8 / RGBA16F (+ radiance, shard) per pixel
//
// Measured motivation (profiles/r01_*): the per-thread megakernel ran primary rays at 19/32
// active lanes but the whole frame at 11/32, because lanes idled while their neighbours traced
// shadow and reflection rays.  Queues keep warps full and let each kernel use few registers.
//
// The sum over a pixel's tree equals the recursive definition (reading 17).  Contributions are
// accumulated in 64-bit fixed point (2^-40; all terms >= 0) so the result does not depend on
// the order in which the atomics land: frames are bit-reproducible.
#include "rt_trace.cuh"

namespace rtb {

#ifndef RT_WAVE_MINB
#define RT_WAVE_MINB 5
#endif

constexpr double ACC_SCALE = 1099511627776.0;   // 2^40

__device__ __forceinline__ void acc_add(unsigned long long* a, float3 c) {
    atomicAdd(&a[0], __double2ull_rn((double)c.x * ACC_SCALE));
    atomicAdd(&a[1], __double2ull_rn((double)c.y * ACC_SCALE));
    atomicAdd(&a[2], __double2ull_rn((double)c.z * ACC_SCALE));
}

// Warp-aggregated append: every lane with `want` gets a distinct slot in [*counter, ...).
__device__ __forceinline__ int append_slot(int* counter, bool want) {
    const unsigned act = __activemask();
    const unsigned m = __ballot_sync(act, want);
    if (!m) return -1;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(counter, __popc(m));
    base = __shfl_sync(act, base, leader);
    return want ? base + __popc(m & ((1u << lane) - 1u)) : -1;
}

template <bool COUNT>
__device__ __forceinline__ void flush_counters(const WaveParams& P, Counters<COUNT>& cnt) {
    if (!COUNT) return;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < RT_NUM_COUNTERS_INTERNAL; ++i) {
        uint32_t v = cnt.c[i];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0 && v) atomicAdd(&P.counters[i], (unsigned long long)v);
    }
}

// ---------------------------------------------------------------- extend: nearest hits
template <bool COUNT, bool BRUTE>
__global__ void __launch_bounds__(256, RT_WAVE_MINB) k_extend(const WaveParams P) {
    extern __shared__ int s_stack[];
    int* const stk = s_stack + threadIdx.x;
    Counters<COUNT> cnt;
    cnt.zero();
    const int n = P.level == 0 ? P.n_work : *P.n_in;
    const int stride = gridDim.x * blockDim.x;
    const int n_pad = (n + 31) & ~31;                        // keep whole warps in the loop
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_pad; i += stride) {
        if (i >= n) continue;
        float3 o, d;
        if (P.level == 0) {
            int eye, px, py;
            if (!map_work(P, i, eye, px, py)) {               // ragged tile padding
                P.hits[i] = make_int4(0, 0, -2, 0);
                continue;
            }
            cnt.add(CNT_PIXELS);
            cnt.add(CNT_PRIMARY);
            const float sx = fmaf(2.0f * (px + 0.5f), 1.0f / P.W, -1.0f) * P.cam.tha;
            const float sy = fmaf(-2.0f * (py + 0.5f), 1.0f / P.H, 1.0f) * P.cam.th;
            d = normalize(P.cam.f + P.cam.r * (sx + P.cam.sigma[eye]) + P.cam.u * sy);
            o = P.cam.eye[eye];
            P.q_in[2 * i] = make_float4(o.x, o.y, o.z, 1.0f);
            P.q_in[2 * i + 1] = make_float4(d.x, d.y, d.z, __int_as_float(i));
        } else {
            o = xyz(P.q_in[2 * i]);
            d = xyz(P.q_in[2 * i + 1]);
        }
        const Hit h = closest_hit<COUNT, BRUTE>(P.sc, o, d, stk, cnt);
        P.hits[i] = make_int4(__float_as_int(h.t), h.slot, h.gid, 0);
    }
    flush_counters(P, cnt);
}

// ---------------------------------------------------------------- shade: local terms + spawn
template <bool COUNT>
__global__ void __launch_bounds__(256) k_shade(const WaveParams P) {
    Counters<COUNT> cnt;
    cnt.zero();
    const DevScene& S = P.sc;
    const int n = P.level == 0 ? P.n_work : *P.n_in;
    const int depth = P.max_depth - P.level;                 // bounces still allowed
    const int stride = gridDim.x * blockDim.x;
    const int n_pad = (n + 31) & ~31;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_pad; i += stride) {
        int4 h = make_int4(0, 0, -2, 0);
        float4 ra = make_float4(0.f, 0.f, 0.f, 0.f), rb = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < n) {
            h = P.hits[i];
            if (h.z != -2) {
                ra = P.q_in[2 * i];
                rb = P.q_in[2 * i + 1];
            }
        }
        const bool live = h.z != -2;
        const int item = __float_as_int(rb.w);
        const float3 o = xyz(ra), d = xyz(rb);
        const float w = ra.w;
        if (live && P.level == 0 && P.prim_id) {             // reading 20: primary hit ID
            int eye, px, py;
            map_work(P, item, eye, px, py);
            P.prim_id[((long long)eye * P.H + py) * P.W + px] = h.z;
        }
        const bool hit = live && h.z >= 0;
        if (live && !hit) {
            cnt.add(CNT_MISSES);
            acc_add(&P.acc[3 * (long long)item], S.background * w);             // S:203 miss
        }
        float3 p = f3(0.f, 0.f, 0.f), nf = f3(0.f, 0.f, 1.f);
        int mat = 0;
        bool front = true;
        if (hit) {
            cnt.add(CNT_SHADE_HITS);
            const float t = __int_as_float(h.x);
            p = fma3(d, t, o);
            float3 ng;
            if (h.y < 0) {
                const int k = ~h.y;
                ng = xyz(__ldg(&S.planes[k]));
                mat = __ldg(&S.plane_mat[k]);
            } else {
                const float4 a = __ldg(&S.prims[3 * h.y]);
                const float4 b = __ldg(&S.prims[3 * h.y + 1]);
                mat = __float_as_int(b.w);
                if (h.z < S.n_spheres) ng = (p - xyz(a)) * (1.0f / b.x);
                else ng = normalize(cross(xyz(b), xyz(__ldg(&S.prims[3 * h.y + 2]))));
            }
            front = dot(d, ng) < 0.0f;
            nf = front ? ng : ng * -1.0f;
            acc_add(&P.acc[3 * (long long)item], (S.ambient * xyz(__ldg(&S.mats[3 * mat]))) * w);
        }
        // one shadow ray per light with n.l > 0 (reading 2), into that light's queue
        for (int j = 0; j < S.n_lights; ++j) {
            bool want = false;
            float3 os = f3(0.f, 0.f, 0.f), sd = f3(0.f, 0.f, 0.f), term = f3(0.f, 0.f, 0.f);
            float dist = 0.f;
            if (hit) {
                cnt.add(CNT_LIGHT_EVALS);
                const float3 Lp = xyz(__ldg(&S.lights[2 * j]));
                const float3 l = normalize(Lp - p);
                const float ndl = dot(nf, l);
                if (ndl > 0.0f) {
                    const float4 m0 = __ldg(&S.mats[3 * mat]);
                    const float3 ks = xyz(__ldg(&S.mats[3 * mat + 1]));
                    const float3 I = xyz(__ldg(&S.lights[2 * j + 1]));
                    const float3 rv = nf * (2.0f * ndl) - l;
                    const float rdv = -dot(rv, d);
                    const float spec = rdv > 0.0f ? __powf(rdv, m0.w) : 0.0f;
                    term = ((xyz(m0) * I) * ndl + (ks * I) * spec) * w;          // reading 3
                    os = fma3(nf, BIAS, p);
                    const float3 sv = Lp - os;
                    dist = sqrtf(dot(sv, sv));
                    sd = sv * (1.0f / dist);
                    want = true;
                    cnt.add(CNT_SHADOW);
                }
            }
            const int slot = append_slot(&P.n_shadow[j], want);
            if (want) {
                if (slot < P.cap_shadow) {
                    float4* e = P.shadow + 3 * ((long long)j * P.cap_shadow + slot);
                    e[0] = make_float4(os.x, os.y, os.z, dist);
                    e[1] = make_float4(sd.x, sd.y, sd.z, __int_as_float(item));
                    e[2] = make_float4(term.x, term.y, term.z, 0.f);
                } else {
                    atomicOr(P.overflow, 1);
                }
            }
        }
        // children (S:193 reflection, reading 5-6 refraction / TIR)
        bool want_t = false, want_r = false;
        float3 td = f3(0.f, 0.f, 0.f), rdir = f3(0.f, 0.f, 0.f);
        float wt = 0.f, wr = 0.f;
        if (hit && depth > 0) {
            const float4 m1 = __ldg(&S.mats[3 * mat + 1]);
            const float4 m2 = __ldg(&S.mats[3 * mat + 2]);
            float kr_eff = m1.w;
            const float kt = m2.x;
            if (kt > 0.0f) {
                const float eta = front ? 1.0f / m2.y : m2.y;
                const float cosi = -dot(d, nf);
                const float kk = 1.0f - eta * eta * (1.0f - cosi * cosi);
                if (kk < 0.0f) {
                    kr_eff += kt;
                } else {
                    td = normalize(d * eta + nf * (eta * cosi - sqrtf(kk)));
                    wt = w * kt;
                    want_t = true;
                    cnt.add(CNT_REFRACTION);
                }
            }
            if (kr_eff > 0.0f) {
                rdir = normalize(d - nf * (2.0f * dot(d, nf)));
                wr = w * kr_eff;
                want_r = true;
                cnt.add(CNT_REFLECTION);
            }
        }
        const int st = append_slot(P.n_out, want_t);
        if (want_t) {
            if (st < P.cap_rays) {
                const float3 to = fma3(nf, -BIAS, p);
                P.q_out[2 * st] = make_float4(to.x, to.y, to.z, wt);
                P.q_out[2 * st + 1] = make_float4(td.x, td.y, td.z, __int_as_float(item));
            } else {
                atomicOr(P.overflow, 1);
            }
        }
        const int sr = append_slot(P.n_out, want_r);
        if (want_r) {
            if (sr < P.cap_rays) {
                const float3 ro = fma3(nf, BIAS, p);
                P.q_out[2 * sr] = make_float4(ro.x, ro.y, ro.z, wr);
                P.q_out[2 * sr + 1] = make_float4(rdir.x, rdir.y, rdir.z, __int_as_float(item));
            } else {
                atomicOr(P.overflow, 1);
            }
        }
    }
    flush_counters(P, cnt);
}

// ---------------------------------------------------------------- occlude: shadow rays
template <bool COUNT, bool BRUTE>
__global__ void __launch_bounds__(256, RT_WAVE_MINB) k_occlude(const WaveParams P) {
    extern __shared__ int s_stack[];
    int* const stk = s_stack + threadIdx.x;
    Counters<COUNT> cnt;
    cnt.zero();
    const int stride = gridDim.x * blockDim.x;
    for (int j = 0; j < P.sc.n_lights; ++j) {                 // one light at a time: coherent batches
        const int n = min(P.n_shadow[j], P.cap_shadow);
        const float4* q = P.shadow + 3 * (long long)j * P.cap_shadow;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
            const float4 a = q[3 * i], b = q[3 * i + 1];
            if (!occluded<COUNT, BRUTE>(P.sc, xyz(a), xyz(b), a.w, stk, cnt))
                acc_add(&P.acc[3 * (long long)__float_as_int(b.w)], xyz(q[3 * i + 2]));
        }
    }
    flush_counters(P, cnt);
}

// ---------------------------------------------------------------- finalize: pack
__global__ void __launch_bounds__(256) k_finalize(const WaveParams P) {
    const int stride = gridDim.x * blockDim.x;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < P.n_work; k += stride) {
        int eye, px, py;
        if (!map_work(P, k, eye, px, py)) continue;
        const unsigned long long* a = P.acc + 3 * (long long)k;
        const float3 c = f3((float)((double)a[0] * (1.0 / ACC_SCALE)), (float)((double)a[1] * (1.0 / ACC_SCALE)),
                            (float)((double)a[2] * (1.0 / ACC_SCALE)));
        if (P.fb[eye]) store_px(P.fb[eye], P.fb_fmt[eye], P.fb_pitch[eye], px, py, c);
        if (P.radiance) P.radiance[((long long)eye * P.H + py) * P.W + px] = make_float4(c.x, c.y, c.z, 0.0f);
        if (P.shard) {
            const long long s = (long long)(k >> 8) * 256 + ((py % TILE) * TILE + (px % TILE));
            if (P.shard_fmt == RT_FORMAT_RGBA8) reinterpret_cast<uint32_t*>(P.shard)[s] = pack_rgba8(c);
            else reinterpret_cast<uint2*>(P.shard)[s] = pack_rgba16f(c);
        }
    }
    if (P.peer_fence) __threadfence_system();                // peer framebuffer stores visible system-wide
}

}  // namespace rtb

using namespace rtb;

template <bool COUNT, bool BRUTE>
static cudaError_t level_impl(const WaveParams& P, int grid, cudaStream_t st) {
    const size_t smem = (size_t)P.stack_entries * 256 * sizeof(int);
    cudaError_t e = cudaFuncSetAttribute(k_extend<COUNT, BRUTE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_occlude<COUNT, BRUTE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_extend<COUNT, BRUTE><<<grid, 256, smem, st>>>(P);
    k_shade<COUNT><<<grid, 256, 0, st>>>(P);
    k_occlude<COUNT, BRUTE><<<grid, 256, smem, st>>>(P);
    return cudaGetLastError();
}

cudaError_t rtb_wave_level(const WaveParams& P, unsigned flags, int grid, cudaStream_t st) {
    const bool count = flags & RT_RENDER_COUNT, brute = flags & RT_RENDER_BRUTE_FORCE;
    if (count && brute) return level_impl<true, true>(P, grid, st);
    if (count) return level_impl<true, false>(P, grid, st);
    if (brute) return level_impl<false, true>(P, grid, st);
    return level_impl<false, false>(P, grid, st);
}

cudaError_t rtb_wave_finalize(const WaveParams& P, int grid, cudaStream_t st) {
    k_finalize<<<grid, 256, 0, st>>>(P);
    return cudaGetLastError();
}

cudaError_t rtb_wave_occupancy(unsigned flags, int stack_entries, int* blocks_per_sm) {
    const bool count = flags & RT_RENDER_COUNT, brute = flags & RT_RENDER_BRUTE_FORCE;
    const void* f = count ? (brute ? (const void*)k_extend<true, true> : (const void*)k_extend<true, false>)
                          : (brute ? (const void*)k_extend<false, true> : (const void*)k_extend<false, false>);
    const size_t smem = (size_t)stack_entries * 256 * sizeof(int);
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, f, 256, smem);
}
