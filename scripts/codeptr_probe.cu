#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void target_kernel(int* out){ out[0]=1; }
__device__ __noinline__ int dfun(int x){ return x*3+1; }
__global__ void probe(unsigned long long* out, int x){
  out[0]=(unsigned long long)(void*)dfun;
  out[1]=(unsigned long long)(void*)target_kernel;
  out[2]=(unsigned long long)(void*)probe;
  int (*fp)(int) = x > 100 ? nullptr : dfun;
  out[3]=fp(x);
}
__global__ void reader(const unsigned int* p, unsigned int* out){ for(int i=0;i<32;i++) out[i]=__ldcg(p+i); }
int main(){
  unsigned long long* d; cudaMalloc(&d, 64); unsigned long long h[4];
  probe<<<1,1>>>(d, 5); cudaError_t e=cudaDeviceSynchronize(); printf("probe %s\n", cudaGetErrorString(e));
  cudaMemcpy(h,d,32,cudaMemcpyDeviceToHost);
  printf("dfun %llx target %llx probe %llx call %llu\n",h[0],h[1],h[2],h[3]);
  cudaPointerAttributes a; e=cudaPointerGetAttributes(&a,(void*)h[1]); printf("attr %s type %d\n", cudaGetErrorString(e), (int)a.type);
  unsigned int* o; cudaMalloc(&o,128); unsigned int ho[32];
  for (int k=0;k<3;k++){
    reader<<<1,1>>>((const unsigned int*)h[k], o); e=cudaDeviceSynchronize(); printf("read %d: %s\n",k,cudaGetErrorString(e));
    if(e) return 0;
    cudaMemcpy(ho,o,128,cudaMemcpyDeviceToHost); for(int i=0;i<16;i++) printf("%08x ", ho[i]); printf("\n");
  }
  return 0;
}
