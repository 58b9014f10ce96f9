#include <cstdio>
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c){
  unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__global__ void k(float* o, float x){ unsigned long long a=__float_as_uint(x), b=a, c=a; for(int i=0;i<4;i++) c=ffma2(a,b,c); o[0]=__uint_as_float((unsigned)c);}
int main(){return 0;}
