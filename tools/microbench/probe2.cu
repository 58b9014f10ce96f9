#include <cstdio>
__global__ void k(const float* __restrict__ in, float* o){
  float s = in[threadIdx.x];
  float2 b = reinterpret_cast<const float2*>(in)[threadIdx.x+64];
  float2 c = reinterpret_cast<const float2*>(in)[threadIdx.x+128];
  float2 b2 = reinterpret_cast<const float2*>(in)[threadIdx.x+192];
  float s2 = in[threadIdx.x+7];
  #pragma unroll
  for(int i=0;i<4;i++){ c = __ffma2_rn(make_float2(s,s), b, c); c = __ffma2_rn(make_float2(s2,s2), make_float2(b2.y,b2.x), c);}
  reinterpret_cast<float2*>(o)[threadIdx.x]=c;
}
int main(){return 0;}
