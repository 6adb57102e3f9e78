#include <cstdio>
#include <cstdlib>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b){u64 r; asm("mov.b64 %0, {%1,%2};":"=l"(r):"f"(a),"f"(b)); return r;}
__device__ __forceinline__ float2 upk(u64 r){float2 v; asm("mov.b64 {%0,%1}, %2;":"=f"(v.x),"=f"(v.y):"l"(r)); return v;}
// variant A: mul as fma(a,b,-0), add as fma(p,1,s)
__device__ __forceinline__ u64 mul2A(u64 a, u64 b){u64 r; asm("fma.rn.f32x2 %0, %1, %2, %3;":"=l"(r):"l"(a),"l"(b),"l"(0x8000000080000000ull)); return r;}
__device__ __forceinline__ u64 add2A(u64 a, u64 b){u64 r; asm("fma.rn.f32x2 %0, %1, %2, %3;":"=l"(r):"l"(a),"l"(0x3f8000003f800000ull),"l"(b)); return r;}
// variant B: plain mul.rn + add.rn
__device__ __forceinline__ u64 mul2B(u64 a, u64 b){u64 r; asm("mul.rn.f32x2 %0, %1, %2;":"=l"(r):"l"(a),"l"(b)); return r;}
__device__ __forceinline__ u64 add2B(u64 a, u64 b){u64 r; asm("add.rn.f32x2 %0, %1, %2;":"=l"(r):"l"(a),"l"(b)); return r;}
// variant C: mul via mul.rn.f32x2, add via two scalar add.rn
__device__ __forceinline__ u64 add2C(u64 a, u64 b){float2 x=upk(a), y=upk(b); return pk(__fadd_rn(x.x,y.x), __fadd_rn(x.y,y.y));}
template<int V> __global__ void k(float2* o, const float2* a, const float2* b, const float2* c, int n){
  int i = blockIdx.x*blockDim.x+threadIdx.x; if(i>=n) return;
  float2 x=a[i], y=b[i], z=c[i];
  u64 X=pk(x.x,x.y), Y=pk(y.x,y.y), Z=pk(z.x,z.y), s;
  // chain of 3 multiply-accumulate terms like the stencil
  if (V==0) { s = add2A(add2A(add2A(Z, mul2A(X,Y)), mul2A(Y,Z)), mul2A(X,Z)); }
  else if (V==1) { s = add2B(add2B(add2B(Z, mul2B(X,Y)), mul2B(Y,Z)), mul2B(X,Z)); }
  else if (V==2) { s = add2C(add2C(add2C(Z, mul2B(X,Y)), mul2B(Y,Z)), mul2B(X,Z)); }
  else {
    float2 r;
    r.x = __fadd_rn(__fadd_rn(__fadd_rn(z.x, __fmul_rn(x.x,y.x)), __fmul_rn(y.x,z.x)), __fmul_rn(x.x,z.x));
    r.y = __fadd_rn(__fadd_rn(__fadd_rn(z.y, __fmul_rn(x.y,y.y)), __fmul_rn(y.y,z.y)), __fmul_rn(x.y,z.y));
    o[i]=r; return;
  }
  o[i]=upk(s);
}
int main(){
  const int n=1<<20; size_t B=n*sizeof(float2);
  float2 *h=(float2*)malloc(3*B), *r[4]; for(int v=0;v<4;v++) r[v]=(float2*)malloc(B);
  srand(1); for(int i=0;i<3*n;i++){ h[i].x=(rand()/(float)RAND_MAX-0.5f)*3; h[i].y=(rand()/(float)RAND_MAX-0.5f)*3; }
  h[0].x = -0.0f; h[n].x = 5.0f; h[2*n].x = -0.0f;
  float2 *d,*o; cudaMalloc(&d,3*B); cudaMalloc(&o,B); cudaMemcpy(d,h,3*B,cudaMemcpyHostToDevice);
  k<0><<<n/256,256>>>(o,d,d+n,d+2*n,n); cudaMemcpy(r[0],o,B,cudaMemcpyDeviceToHost);
  k<1><<<n/256,256>>>(o,d,d+n,d+2*n,n); cudaMemcpy(r[1],o,B,cudaMemcpyDeviceToHost);
  k<2><<<n/256,256>>>(o,d,d+n,d+2*n,n); cudaMemcpy(r[2],o,B,cudaMemcpyDeviceToHost);
  k<3><<<n/256,256>>>(o,d,d+n,d+2*n,n); cudaMemcpy(r[3],o,B,cudaMemcpyDeviceToHost);
  for (int v=0; v<3; v++){ int diff=0; for(int i=0;i<n;i++) diff += (memcmp(&r[v][i].x,&r[3][i].x,4)!=0) + (memcmp(&r[v][i].y,&r[3][i].y,4)!=0);
    printf("variant %d vs scalar: %d of %d differ\n", v, diff, 2*n); }
  return 0;
}
