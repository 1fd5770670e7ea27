// common.cuh -- shared device types and helpers for the sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#define VRP_FULL_MASK 0xffffffffu

// Device view of an uploaded instance (instance.py:82-156).
struct DevInstance {
    int32_t n, m, k, W;       // W = n + 1 (row pitch of d)
    const double *d;          // (n+1)^2 fp64
    const int32_t *d32;       // same values as int32 when `integral`, else null
    const int32_t *d32t;      // its transpose (d32t[b*W + a] = d[a][b]) when `integral`, else null
    const double *p;          // n+1 fp64
    const int32_t *p32;       // same values as int32 when `integral`, else null
    int32_t integral;         // every d and p entry is an integer in [0, 2^31)
};

// op code = 2*(c-1) + kind  (brkga.py:73-75)
__device__ __forceinline__ int op_customer(int op) { return (op >> 1) + 1; }
__device__ __forceinline__ bool op_is_pick(int op) { return op & 1; }

// Travel time d[a][b] as fp64.  The int32 table (integral instances) gives the
// identical double value with half the L2 sector footprint per row.
template <bool INTD>
__device__ __forceinline__ double dist(const DevInstance &I, int a, int b) {
    const uint32_t idx = (uint32_t)a * (uint32_t)I.W + (uint32_t)b;  // n <= 8192: W^2 < 2^27
    if (INTD) return (double)__ldg(I.d32 + idx);
    return __ldg(I.d + idx);
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

__device__ __forceinline__ double warp_max(double x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        double y = __shfl_xor_sync(VRP_FULL_MASK, x, o);
        x = y > x ? y : x;
    }
    return x;
}

__device__ __forceinline__ int warp_sum(int x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(VRP_FULL_MASK, x, o);
    return x;
}

// streaming (read-once) load: keep the candidate stream from evicting the
// L2-resident distance matrix.
template <typename T>
__device__ __forceinline__ T load_stream(const T *p) { return __ldcs(p); }

// host-side launch helpers (capi.cu)
struct LaunchShape {
    int warps_per_block;
    int blocks;
    size_t smem_bytes;
};

// Launch plans (block shape, dynamic shared memory, the MaxDynamicSharedMemory
// attribute) computed once per (device, key) and kept per device -- the
// attribute is per device -- under a mutex, so one process may drive several
// GPUs from several threads.  make(plan) returns 0 or an error code.
constexpr int VRP_MAX_DEVICES = 64;
template <typename Plan>
struct PlanCache {
    std::mutex mu;
    int64_t key[VRP_MAX_DEVICES];
    bool valid[VRP_MAX_DEVICES] = {};
    Plan plan[VRP_MAX_DEVICES];

    template <typename F>
    int get(int64_t k, Plan &out, F make) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= VRP_MAX_DEVICES) return -1;
        std::lock_guard<std::mutex> lock(mu);
        if (!valid[dev] || key[dev] != k) {
            valid[dev] = false;
            const int rc = make(plan[dev]);
            if (rc) return rc;
            key[dev] = k;
            valid[dev] = true;
        }
        out = plan[dev];
        return 0;
    }
};
