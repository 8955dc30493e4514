// stream_copy_ref.cu -- the achievable HBM rate of the C5 access pattern with no
// arithmetic: read 13 fp32 arrays (r, p, E, B, weight), write 7 (r, p, gamma),
// 128-bit accesses, the same grid-stride shape as k_stream_soa_vec.  The push
// kernel's measured GB/s divided by this kernel's GB/s is its efficiency against
// its own access pattern (tuning evidence only; not part of libboris).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/scr stream_copy_ref.cu && /tmp/scr
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float4 ldg(const float *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void stg(float *p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}

struct Ptrs {
    const float *in[13];
    float *out[7];
};

__global__ void __launch_bounds__(256) k_copy_pattern(Ptrs p, long long groups) {
    for (long long g = (long long)blockIdx.x * 256 + threadIdx.x; g < groups;
         g += (long long)gridDim.x * 256) {
        float4 v[13];
#pragma unroll
        for (int a = 0; a < 13; ++a) v[a] = ldg(p.in[a] + 4 * g);
        float4 o[7];
#pragma unroll
        for (int a = 0; a < 7; ++a) {  // cheap mix so no load is dead
            o[a].x = v[a].x + v[a + 6].x;
            o[a].y = v[a].y + v[a + 6].y;
            o[a].z = v[a].z + v[a + 6].z;
            o[a].w = v[a].w + v[a + 6].w;
        }
#pragma unroll
        for (int a = 0; a < 7; ++a) stg(p.out[a] + 4 * g, o[a]);
    }
}

int main() {
    for (long long n : {100000000LL, 800000000LL}) {
        Ptrs p;
        float *buf[20];
        for (int a = 0; a < 20; ++a) {
            if (cudaMalloc(&buf[a], n * sizeof(float)) != cudaSuccess) {
                printf("alloc failed\n");
                return 1;
            }
            cudaMemset(buf[a], 0, n * sizeof(float));
        }
        for (int a = 0; a < 13; ++a) p.in[a] = buf[a];
        for (int a = 0; a < 7; ++a) p.out[a] = buf[13 + a];
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        const long long groups = n / 4;
        long long blocks = (groups + 255) / 256, cap = (long long)sms * 8 * 4;
        const unsigned grid = (unsigned)(blocks < cap ? blocks : cap);
        for (int i = 0; i < 5; ++i) k_copy_pattern<<<grid, 256>>>(p, groups);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        const int iters = n > 200000000LL ? 100 : 800;
        cudaEventRecord(a);
        for (int i = 0; i < iters; ++i) k_copy_pattern<<<grid, 256>>>(p, groups);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        ms /= iters;
        printf("{\"exp\": \"copy_pattern_13r_7w\", \"n\": %lld, \"ms\": %.5f, \"gbs\": %.1f}\n", n, ms,
               80.0 * n / (ms * 1e-3) / 1e9);
        for (int i = 0; i < 20; ++i) cudaFree(buf[i]);
    }
    return 0;
}
