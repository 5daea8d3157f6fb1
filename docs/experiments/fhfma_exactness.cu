// Is the sm_100 mixed-precision FMA (PTX fma.rn.f32.f16, SASS FHFMA) exactly h*s + k rounded once?
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/fhfma docs/experiments/fhfma_exactness.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_fp16.h>
__global__ void k(const unsigned short* h, const unsigned short* s, const float* c, float* out, float* out2, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float r, r2;
    asm("{.reg .f16 a, b; mov.b16 a, %1; mov.b16 b, %2; fma.rn.f32.f16 %0, a, b, %3;}" : "=f"(r) : "h"(h[i]), "h"(s[i]), "f"(c[i]));
    asm("{.reg .f16 a; mov.b16 a, %1; add.rn.f32.f16 %0, a, %2;}" : "=f"(r2) : "h"(h[i]), "f"(c[i]));
    out[i] = r;
    out2[i] = r2;
}
int main() {
    const int n = 1 << 20;
    unsigned short *h, *s; float *c, *o, *o2;
    cudaMallocManaged(&h, n * 2); cudaMallocManaged(&s, n * 2); cudaMallocManaged(&c, n * 4);
    cudaMallocManaged(&o, n * 4); cudaMallocManaged(&o2, n * 4);
    srand(1);
    for (int i = 0; i < n; ++i) {
        float hv = (float)(rand() % 16384) + (rand() % 1024) / 1024.0f;
        h[i] = __half_as_ushort(__float2half_rn(hv));
        int e = -14 + rand() % 10;
        s[i] = __half_as_ushort(__float2half_rn(ldexpf(1.0f, e)));
        c[i] = ((rand() / (float)RAND_MAX) - 0.5f) * 8.0f;
    }
    k<<<(n + 255) / 256, 256>>>(h, s, c, o, o2, n);
    cudaDeviceSynchronize();
    int bad = 0, bad2 = 0; double worst = 0, worst2 = 0;
    for (int i = 0; i < n; ++i) {
        double hv = __half2float(__ushort_as_half(h[i])), sv = __half2float(__ushort_as_half(s[i]));
        float ref = (float)(hv * sv + (double)c[i]);       // exact product, one rounding (double then float ~ RN)
        float ref2 = (float)(hv + (double)c[i]);
        if (ref != o[i]) { ++bad; worst = fmax(worst, fabs((double)o[i] - ref) / fmax(fabs(ref), 1e-30)); }
        if (ref2 != o2[i]) { ++bad2; worst2 = fmax(worst2, fabs((double)o2[i] - ref2) / fmax(fabs(ref2), 1e-30)); }
    }
    printf("fma.rn.f32.f16: %d / %d differ from h*s+k rounded once (worst rel %.3g)\n", bad, n, worst);
    printf("add.rn.f32.f16: %d / %d differ from h+k rounded once (worst rel %.3g)\n", bad2, n, worst2);
    return 0;
}
