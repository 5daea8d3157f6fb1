// rt_probe.cu -- B0 machine-ceiling microbenchmarks (SURVEY §8(d) "verify in B0"): the
// denominators the trace kernel's roofline and its SASS-derived ceiling are quoted against.
//
// Every probe runs one CTA of 1024 threads (32 warps, 8 per SMSP) on every SM and times its
// own body with the SM cycle counter between two CTA barriers, so each result is per SM per
// clock -- independent of the clock the GPU happens to run at -- and the event-timed duration of
// a long FFMA run gives the clock itself.
//   ffma  (3 registers)  x = fma(x, y, z), y and z registers: the form the slab test uses
//   ffma2                packed FP32 FMA on register pairs (sm_100 FFMA2, the slab test's form)
//   fmnmx / fmnmx3       2- and 3-input FP32 max on the ALU pipe (the box tests' min/max)
//   ldg  (L1 hit)        128-bit loads of a 16 KB block that stays in L1
//   lds                  128-bit shared-memory loads, conflict free
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "rt_internal.h"

namespace rtb {

constexpr int PROBE_THREADS = 1024;

struct ProbeOut {
    unsigned long long cycles;  // SM cycles of the timed body (thread 0 of the CTA)
    float sink;
};

__device__ __forceinline__ void probe_end(ProbeOut* out, unsigned long long t0, float v) {
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x].cycles = t1 - t0;
    if (v == 1234.5f) out[blockIdx.x].sink = v;          // keeps the chains alive
}

// 8 independent chains per thread, 16 unrolled steps per iteration: 128 FFMA per iteration
__global__ void __launch_bounds__(PROBE_THREADS) k_probe_ffma(ProbeOut* out, int iters, float y0, float z0) {
    float x[8], y[8], z[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        x[k] = threadIdx.x + k;
        y[k] = y0 + 1e-7f * k;
        z[k] = z0 * (k + 1);
    }
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], y[(k + j) & 7], z[(k + 3 * j) & 7]);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    probe_end(out, t0, s);
}

// 8 independent float2 chains: 128 FFMA2 (256 FMA) per iteration
__global__ void __launch_bounds__(PROBE_THREADS) k_probe_ffma2(ProbeOut* out, int iters, float y0, float z0) {
    float2 x[8], y[8], z[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        x[k] = make_float2(threadIdx.x + k, threadIdx.x - k);
        y[k] = make_float2(y0 + 1e-7f * k, y0 - 1e-7f * k);
        z[k] = make_float2(z0 * (k + 1), z0 * (k + 2));
    }
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = __ffma2_rn(x[k], y[(k + j) & 7], z[(k + 3 * j) & 7]);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k].x + x[k].y;
    probe_end(out, t0, s);
}

// 8 independent max chains (inline PTX so nothing folds): 128 FMNMX (or FMNMX3) per iteration
template <bool THREE>
__global__ void __launch_bounds__(PROBE_THREADS) k_probe_fmnmx(ProbeOut* out, int iters, float y0) {
    float x[8], y[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        x[k] = -1e30f + threadIdx.x + k;
        y[k] = y0 + k;
    }
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (THREE)
                    asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(x[k]) : "f"(y[(k + j) & 7]), "f"(y[(k + 5 * j + 1) & 7]));
                else
                    asm volatile("max.f32 %0, %0, %1;" : "+f"(x[k]) : "f"(y[(k + j) & 7]));
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    probe_end(out, t0, s);
}

// L1-resident 128-bit loads: each warp streams through its CTA's 16 KB block (CTA-private, so it
// stays in L1 after the first pass); 8 independent loads in flight per thread per step
__global__ void __launch_bounds__(PROBE_THREADS) k_probe_ldg(ProbeOut* out, const uint4* __restrict__ buf, int iters) {
    const uint4* b = buf + (size_t)blockIdx.x * 1024;        // 16 KB per CTA
    uint32_t acc = 0;
    for (int k = threadIdx.x; k < 1024; k += PROBE_THREADS) acc ^= __ldg(&b[k]).x;   // warm L1
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint4 v = __ldg(&b[(threadIdx.x + j * 128 + i * 32) & 1023]);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    }
    probe_end(out, t0, (float)(acc & 1u) + 1234.5f * (acc == 0x9e3779b9u));
}

// conflict-free 128-bit shared loads
__global__ void __launch_bounds__(PROBE_THREADS) k_probe_lds(ProbeOut* out, int iters) {
    __shared__ uint4 s[2048];                               // 32 KB
    for (int k = threadIdx.x; k < 2048; k += PROBE_THREADS) s[k] = make_uint4(k, k * 3, k * 5, k * 7);
    uint32_t acc = 0;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint4 v = s[(threadIdx.x + j * 256 + i * 32) & 2047];
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    }
    probe_end(out, t0, (float)(acc & 1u) + 1234.5f * (acc == 0x9e3779b9u));
}

}  // namespace rtb

using namespace rtb;

namespace {

// median over CTAs of (work per CTA) / cycles
double per_sm_per_clk(const std::vector<ProbeOut>& o, double work_per_cta) {
    std::vector<double> r;
    for (const auto& x : o)
        if (x.cycles) r.push_back(work_per_cta / (double)x.cycles);
    if (r.empty()) return 0.0;
    std::sort(r.begin(), r.end());
    return r[r.size() / 2];
}

}  // namespace

cudaError_t rtb_probe_ceilings(int num_sms, cudaStream_t st, double out[RT_NUM_CEILINGS]) {
    ProbeOut* d = nullptr;
    uint4* buf = nullptr;
    cudaError_t e = cudaMalloc(&d, sizeof(ProbeOut) * num_sms);
    if (e == cudaSuccess) e = cudaMalloc(&buf, (size_t)num_sms * 1024 * sizeof(uint4));
    if (e == cudaSuccess) e = cudaMemsetAsync(buf, 1, (size_t)num_sms * 1024 * sizeof(uint4), st);
    std::vector<ProbeOut> h(num_sms);
    cudaEvent_t a = nullptr, b = nullptr;
    if (e == cudaSuccess) e = cudaEventCreate(&a);
    if (e == cudaSuccess) e = cudaEventCreate(&b);
    const double T = PROBE_THREADS;
    auto run = [&](auto launch, double work_per_cta, int slot, bool clock) -> cudaError_t {
        cudaError_t r = cudaMemsetAsync(d, 0, sizeof(ProbeOut) * num_sms, st);
        if (r == cudaSuccess) { launch(); r = cudaGetLastError(); }                        // warm-up
        if (r == cudaSuccess) r = cudaEventRecord(a, st);
        if (r == cudaSuccess) { launch(); r = cudaGetLastError(); }
        if (r == cudaSuccess) r = cudaEventRecord(b, st);
        if (r == cudaSuccess) r = cudaMemcpyAsync(h.data(), d, sizeof(ProbeOut) * num_sms, cudaMemcpyDeviceToHost, st);
        if (r == cudaSuccess) r = cudaStreamSynchronize(st);
        if (r != cudaSuccess) return r;
        out[slot] = per_sm_per_clk(h, work_per_cta);
        if (clock) {            // SM clock = cycles of the body / event time (long body: launch cost negligible)
            float ms = 0.f;
            cudaEventElapsedTime(&ms, a, b);
            std::vector<double> cy;
            for (auto& x : h) cy.push_back((double)x.cycles);
            std::sort(cy.begin(), cy.end());
            out[RT_CEIL_SM_MHZ] = ms > 0 ? cy.back() / (ms * 1e-3) / 1e6 : 0.0;
        }
        return cudaSuccess;
    };
    const int it = 4096;
    if (e == cudaSuccess)
        e = run([&] { k_probe_ffma<<<num_sms, PROBE_THREADS, 0, st>>>(d, it, 1.0000001f, 1e-7f); }, 2.0 * 128 * it * T,
                RT_CEIL_FFMA_FLOP_CLK, true);
    if (e == cudaSuccess)
        e = run([&] { k_probe_ffma2<<<num_sms, PROBE_THREADS, 0, st>>>(d, it, 1.0000001f, 1e-7f); }, 4.0 * 128 * it * T,
                RT_CEIL_FFMA2_FLOP_CLK, false);
    if (e == cudaSuccess)
        e = run([&] { k_probe_fmnmx<false><<<num_sms, PROBE_THREADS, 0, st>>>(d, it, 0.5f); }, 128.0 * it * T,
                RT_CEIL_FMNMX_CLK, false);
    if (e == cudaSuccess)
        e = run([&] { k_probe_fmnmx<true><<<num_sms, PROBE_THREADS, 0, st>>>(d, it, 0.5f); }, 128.0 * it * T,
                RT_CEIL_FMNMX3_CLK, false);
    if (e == cudaSuccess)
        e = run([&] { k_probe_ldg<<<num_sms, PROBE_THREADS, 0, st>>>(d, buf, it); }, 16.0 * 8 * it * T,
                RT_CEIL_L1_BYTES_CLK, false);
    if (e == cudaSuccess)
        e = run([&] { k_probe_lds<<<num_sms, PROBE_THREADS, 0, st>>>(d, it); }, 16.0 * 8 * it * T,
                RT_CEIL_SMEM_BYTES_CLK, false);
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
    if (d) cudaFree(d);
    if (buf) cudaFree(buf);
    return e;
}
