#include <cstdio>
#include <cuda_runtime.h>
int main(){cudaDeviceProp p; cudaGetDeviceProperties(&p,0); printf("persistingL2CacheMaxSize %d MB, accessPolicyMaxWindowSize %d MB, l2 %d MB\n", p.persistingL2CacheMaxSize>>20, p.accessPolicyMaxWindowSize>>20, p.l2CacheSize>>20); return 0;}
