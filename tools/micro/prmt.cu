#include <cstdio>
__global__ void k(unsigned a, unsigned b, unsigned* out) {
    unsigned r;
    asm("prmt.b32 %0, %1, %2, 0x44fb;" : "=r"(r) : "r"(a), "r"(b));
    out[0] = r;
}
int main() {
    unsigned* d; cudaMalloc(&d, 4);
    unsigned tests[4][2] = {{0x80000000u, 0x12345678u}, {0x7fffffffu, 0x80345678u}, {0xbff00000u, 0xbff00000u}, {0x3ff00000u, 0x3ff00000u}};
    for (auto& t : tests) { k<<<1, 1>>>(t[0], t[1], d); unsigned h; cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost); printf("a=%08x b=%08x -> %08x  &0x110 = %03x\n", t[0], t[1], h, h & 0x110); }
}
