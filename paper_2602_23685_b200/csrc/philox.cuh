// philox.cuh -- numpy's Generator(Philox) on the device (numpy/random/src/philox,
// distributions.c): Philox4x64-10 with a pre-incremented 256-bit counter, a
// 4-word output buffer, random() = (u64 >> 11) * 2^-53, and integers(n) via
// 32-bit Lemire over a persistent u32 half-buffer.  Two access styles:
//   stream_u64(S, q)  -- counter-based random access (parallel kernels, K4)
//   PhiloxGen         -- sequential draws exactly like the Python object (K5)
#pragma once
#include <stdint.h>

#include "../../include/vrp_rpd.h"

__device__ __forceinline__ void philox_block(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                                             uint64_t k0, uint64_t k1, uint64_t out[4]) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += 0x9E3779B97F4A7C15ULL; k1 += 0xBB67AE8584CAA73BULL; }
        const uint64_t lo0 = 0xD2E7470EE14C6C93ULL * c0, hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, c0);
        const uint64_t lo1 = 0xCA5A826395121157ULL * c2, hi1 = __umul64hi(0xCA5A826395121157ULL, c2);
        const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// 128-bit counter + j (j >= 0)
__device__ __forceinline__ void ctr_add(const uint64_t *ctr, uint64_t j, uint64_t out[4]) {
    uint64_t a = ctr[0] + j;
    uint64_t carry = a < ctr[0];
    out[0] = a;
    uint64_t b = ctr[1] + carry; carry = carry && b == 0; out[1] = b;
    uint64_t c = ctr[2] + carry; carry = carry && c == 0; out[2] = c;
    out[3] = ctr[3] + carry;
}

// q-th u64 of the stream that starts at state S (numpy philox_next semantics)
__device__ __forceinline__ uint64_t stream_u64(const vrp_philox &S, uint64_t q) {
    const uint64_t head = 4 - (uint64_t)S.buffer_pos;
    if (q < head) return S.buffer[S.buffer_pos + q];
    const uint64_t qq = q - head;
    uint64_t c[4], out[4];
    ctr_add(S.ctr, 1 + qq / 4, c);
    philox_block(c[0], c[1], c[2], c[3], S.key[0], S.key[1], out);
    return out[qq & 3];
}

__device__ __forceinline__ double u64_to_double(uint64_t x) {
    return (double)(x >> 11) * (1.0 / 9007199254740992.0);
}


// Sequential generator: a register copy of the numpy state.
struct PhiloxGen {
    vrp_philox s;

    __device__ __forceinline__ uint64_t next64() {
        if (s.buffer_pos < 4) return s.buffer[s.buffer_pos++];
        uint64_t c[4];
        ctr_add(s.ctr, 1, c);
        for (int j = 0; j < 4; ++j) s.ctr[j] = c[j];
        philox_block(c[0], c[1], c[2], c[3], s.key[0], s.key[1], s.buffer);
        s.buffer_pos = 1;
        return s.buffer[0];
    }
    __device__ __forceinline__ uint32_t next32() {
        if (s.has_uint32) {
            s.has_uint32 = 0;
            return s.uinteger;
        }
        const uint64_t x = next64();
        s.has_uint32 = 1;
        s.uinteger = (uint32_t)(x >> 32);
        return (uint32_t)x;
    }
    __device__ __forceinline__ double next_double() { return u64_to_double(next64()); }
    // Generator.integers(0, n), 1 <= n < 2^32
    __device__ __forceinline__ uint32_t integers(uint32_t n) {
        if (n <= 1) return 0;
        uint64_t m = (uint64_t)next32() * n;
        uint32_t left = (uint32_t)m;
        if (left < n) {
            const uint32_t thresh = (0u - n) % n;
            while (left < thresh) {
                m = (uint64_t)next32() * n;
                left = (uint32_t)m;
            }
        }
        return (uint32_t)(m >> 32);
    }
};
