#include <cstdio>
__device__ __forceinline__ float2 add2(float2 a, float2 b){ return __ffma2_rn(a, make_float2(1.f,1.f), b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b){ return __ffma2_rn(a, b, make_float2(-0.f,-0.f)); }
__global__ void k(float2* a, const float2* b, const float2* c, int n){
  int i = blockIdx.x*blockDim.x+threadIdx.x; if(i>=n) return;
  float2 x=a[i], y=b[i], z=c[i];
  float2 r = mul2(x, y);
  r = add2(r, z);
  float2 r2 = __fadd2_rn(__fmul2_rn(x, y), z);
  float s = __fadd_rn(__fmul_rn(x.x, y.x), z.x);
  a[i] = r; a[i+n] = r2; a[i+2*n] = make_float2(s, s);
}
int main(){
  float2 h[3] = {{1.0f+0x1p-12f, 1.0f+0x1p-12f},{1.0f+0x1p-12f,1.0f+0x1p-12f},{-1.0f,-1.0f}};
  float2 *d; cudaMalloc(&d, sizeof(float2)*3);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  k<<<1,1>>>(d, d+1, d+2, 1);
  float2 o[3]; cudaMemcpy(o, d, sizeof(o), cudaMemcpyDeviceToHost);
  printf("fma-emulated %a  intrinsic2 %a  scalar %a  (unfused expect 0x1p-11, fused 0x1.002p-11)\n", o[0].x, o[1].x, o[2].x);
}
