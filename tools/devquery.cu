#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* o){ o[threadIdx.x] = __dmul_rn(2.0, threadIdx.x); }
int main(){
  cudaDeviceProp p; cudaGetDeviceProperties(&p,0);
  printf("name=%s sms=%d l2=%d smemPerBlockOptin=%zu smemPerSM=%zu regsPerSM=%d clock=%d memclk=%d busw=%d cc=%d.%d\n", p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, p.sharedMemPerMultiprocessor, p.regsPerMultiprocessor, p.clockRate, p.memoryClockRate, p.memoryBusWidth, p.major, p.minor);
  float* d; cudaMalloc(&d, 1024); k<<<1,32>>>(d); float h[32]; cudaMemcpy(h,d,128,cudaMemcpyDeviceToHost);
  printf("kernel ok %f err=%s\n", h[5], cudaGetErrorString(cudaGetLastError()));
}
