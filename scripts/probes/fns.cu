// Semantics check of __fns / __reduce_or_sync with disjoint lane groups.
#include <cstdio>
__global__ void k(unsigned *out) {
    const unsigned masks[3] = {0xB6u, 0x80000001u, 0x0u};
    int lane = threadIdx.x;
    if (lane < 12) {
        unsigned m = masks[lane / 4];
        out[lane] = __fns(m, 0, (lane % 4) + 1);  // n-th set bit, n = 1..4
    }
    // groups of 6 lanes: lanes 0-5, 6-11, ..., 24-29; 30, 31 alone
    int g = lane / 6;
    unsigned gm = g < 5 ? (0x3Fu << (g * 6)) : (1u << lane);
    unsigned v = 1u << (lane % 6 + g);
    unsigned r = __reduce_or_sync(gm, v);
    out[32 + lane] = r;
}
int main() {
    unsigned *d, h[64];
    cudaMalloc(&d, 256);
    k<<<1, 32>>>(d);
    cudaMemcpy(h, d, 256, cudaMemcpyDeviceToHost);
    printf("fns(0xB6,0,n) n=1..4: %u %u %u %u (set bits 1,2,4,5,7)\n", h[0], h[1], h[2], h[3]);
    printf("fns(0x80000001,0,n): %u %u %u %u\n", h[4], h[5], h[6], h[7]);
    printf("fns(0,0,n): %u %u %u %u\n", h[8], h[9], h[10], h[11]);
    for (int l = 0; l < 32; ++l) printf("%x ", h[32 + l]);
    printf("\n");
    return 0;
}
