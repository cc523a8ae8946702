#include <cstdio>
#include <cstdint>
__global__ void k(int* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    if (threadIdx.x == 0) out[blockIdx.x] = (int)(static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)));
}
int main() {
    int* d; cudaMalloc(&d, 64 * 4);
    for (int bytes : {1024, 100000, 232448}) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        k<<<4, 128, bytes>>>(d);
        int h[4]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("dyn %d: base %d %d (mod 1024 = %d) err=%s\n", bytes, h[0], h[1], h[0] % 1024, cudaGetErrorString(cudaGetLastError()));
    }
}
