// Microbenchmarks for the ALU ceilings of the regression path on B200 (sm_100a):
// fp64 add/fma/mul, f32<->f64 conversions, shared-memory atomics (spread / hot / windowed),
// and plain HBM streaming read+write. Prints one line per measurement.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__global__ void k_dfma(double* out, int iters, double a, double b){
  double x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for(int i=0;i<iters;i++){
    x0=fma(x0,a,b); x1=fma(x1,a,b); x2=fma(x2,a,b); x3=fma(x3,a,b);
    x4=fma(x4,a,b); x5=fma(x5,a,b); x6=fma(x6,a,b); x7=fma(x7,a,b);
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void k_dadd(double* out, int iters, double a){
  double x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for(int i=0;i<iters;i++){
    x0=__dadd_rn(x0,a); x1=__dadd_rn(x1,a); x2=__dadd_rn(x2,a); x3=__dadd_rn(x3,a);
    x4=__dadd_rn(x4,a); x5=__dadd_rn(x5,a); x6=__dadd_rn(x6,a); x7=__dadd_rn(x7,a);
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
// f32 -> f64 -> f32 round trips: 2 conversions per step per chain
__global__ void k_cvt(float* out, int iters){
  float x0=threadIdx.x*1.1f, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for(int i=0;i<iters;i++){
    x0=__double2float_rn((double)x0*1.0000001); x1=__double2float_rn((double)x1*1.0000001);
    x2=__double2float_rn((double)x2*1.0000001); x3=__double2float_rn((double)x3*1.0000001);
    x4=__double2float_rn((double)x4*1.0000001); x5=__double2float_rn((double)x5*1.0000001);
    x6=__double2float_rn((double)x6*1.0000001); x7=__double2float_rn((double)x7*1.0000001);
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
// same body without the conversions but with the dmul (to subtract)
__global__ void k_dmul_only(double* out, int iters){
  double x0=threadIdx.x*1.1, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for(int i=0;i<iters;i++){
    x0=x0*1.0000001; x1=x1*1.0000001; x2=x2*1.0000001; x3=x3*1.0000001;
    x4=x4*1.0000001; x5=x5*1.0000001; x6=x6*1.0000001; x7=x7*1.0000001;
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
// int -> double conversions (I2F.F64)
__global__ void k_i2d(double* out, int iters){
  int a=threadIdx.x; double acc0=0,acc1=0,acc2=0,acc3=0;
  for(int i=0;i<iters;i++){
    acc0+= (double)(a+i); acc1+=(double)(a-i); acc2+=(double)(a^i); acc3+=(double)(a|i);
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=acc0+acc1+acc2+acc3;
}
// shared-memory atomics: mode 0 spread (lane-distinct banks), 1 hot (all same bin), 2 pseudo-random within 8192 bins
__global__ void k_atoms(unsigned* out, int iters, int mode){
  __shared__ unsigned h[8192];
  for(int i=threadIdx.x;i<8192;i+=blockDim.x) h[i]=0;
  __syncthreads();
  unsigned s = threadIdx.x*2654435761u + blockIdx.x;
  for(int i=0;i<iters;i++){
    unsigned bin;
    if(mode==0) bin = (threadIdx.x + i*32) & 8191;
    else if(mode==1) bin = 4096;
    else { s = s*1664525u+1013904223u; bin = 4096 + ((int)((s>>16)&511) - 256); }
    atomicAdd(&h[bin],1u);
  }
  __syncthreads();
  unsigned acc=0; for(int i=threadIdx.x;i<8192;i+=blockDim.x) acc+=h[i];
  atomicAdd(out,acc);
}
// hot-bin with warp aggregation via match_any
__global__ void k_atoms_match(unsigned* out, int iters, int mode){
  __shared__ unsigned h[8192];
  for(int i=threadIdx.x;i<8192;i+=blockDim.x) h[i]=0;
  __syncthreads();
  unsigned s = threadIdx.x*2654435761u + blockIdx.x;
  for(int i=0;i<iters;i++){
    unsigned bin;
    if(mode==1) bin = 4096;
    else { s = s*1664525u+1013904223u; bin = 4096 + ((int)((s>>16)&511) - 256); }
    unsigned m = __match_any_sync(0xffffffffu, bin);
    int leader = __ffs(m)-1;
    if((threadIdx.x&31)==leader) atomicAdd(&h[bin],(unsigned)__popc(m));
  }
  __syncthreads();
  unsigned acc=0; for(int i=threadIdx.x;i<8192;i+=blockDim.x) acc+=h[i];
  atomicAdd(out,acc);
}
__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x, st=(size_t)gridDim.x*blockDim.x;
  for(; i<n; i+=st) b[i]=a[i];
}
__global__ void k_read(const float4* __restrict__ a, float* out, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x, st=(size_t)gridDim.x*blockDim.x;
  float acc=0; for(; i<n; i+=st){ float4 v=a[i]; acc+=v.x+v.y+v.z+v.w; }
  if(acc==123.f) out[0]=acc;
}
template<class F> float timeit(F f, int reps){
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); for(int r=0;r<reps;r++) f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms,a,b); return ms/reps;
}
int main(){
  int dev=0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,dev));
  int sms=p.multiProcessorCount; int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("device %s sms %d clock_khz %d l2 %d\n", p.name, sms, clk, p.l2CacheSize);
  double* dout; CK(cudaMalloc(&dout, 1<<26)); unsigned* uout; CK(cudaMalloc(&uout,64));
  int blocks=sms*8, thr=256, iters=4096;
  double ops = (double)blocks*thr*iters*8;
  float ms = timeit([&]{k_dfma<<<blocks,thr>>>(dout,iters,1.0000001,1e-9);},5);
  printf("dfma  lanes/clk/SM @%.0fMHz-equiv: ops/s=%.3e  per-SM-per-ns=%.2f\n", clk/1e3, ops/(ms*1e-3), ops/(ms*1e-3)/sms/1e9);
  ms = timeit([&]{k_dadd<<<blocks,thr>>>(dout,iters,1e-9);},5);
  printf("dadd  ops/s=%.3e per-SM-per-ns=%.2f\n", ops/(ms*1e-3), ops/(ms*1e-3)/sms/1e9);
  ms = timeit([&]{k_dmul_only<<<blocks,thr>>>(dout,iters);},5);
  printf("dmul  ops/s=%.3e per-SM-per-ns=%.2f\n", ops/(ms*1e-3), ops/(ms*1e-3)/sms/1e9);
  float ms2 = timeit([&]{k_cvt<<<blocks,thr>>>((float*)dout,iters);},5);
  printf("cvt-roundtrip (2 cvt + 1 dmul per step) steps/s=%.3e per-SM-per-ns=%.2f -> cvt/SM/ns approx %.2f\n", ops/(ms2*1e-3), ops/(ms2*1e-3)/sms/1e9, 2*ops/((ms2-ms)*1e-3)/sms/1e9);
  ms = timeit([&]{k_i2d<<<blocks,thr>>>(dout,iters);},5);
  printf("i2d (4 cvt+4 dadd per it) its/s per SM per ns=%.3f\n", (double)blocks*thr*iters*4/(ms*1e-3)/sms/1e9);
  for(int mode=0;mode<3;mode++){
    double aops=(double)blocks*thr*iters;
    ms = timeit([&]{k_atoms<<<blocks,thr>>>(uout,iters,mode);},3);
    printf("atoms mode %d (0 spread,1 hot,2 rand512): atom/SM/ns=%.3f\n", mode, aops/(ms*1e-3)/sms/1e9);
  }
  for(int mode=1;mode<3;mode++){
    double aops=(double)blocks*thr*iters;
    ms = timeit([&]{k_atoms_match<<<blocks,thr>>>(uout,iters,mode);},3);
    printf("atoms+match mode %d: elem/SM/ns=%.3f\n", mode, aops/(ms*1e-3)/sms/1e9);
  }
  size_t n = (size_t)1<<30; float4 *a,*b; CK(cudaMalloc(&a,n*4)); CK(cudaMalloc(&b,n*4)); cudaMemset(a,0,n*4);
  size_t n4=n/4;
  ms = timeit([&]{k_copy<<<sms*4,512>>>(a,b,n4);},10);
  printf("copy 4GiB: %.1f GB/s (r+w)\n", 2.0*n*4/(ms*1e-3)/1e9);
  ms = timeit([&]{k_read<<<sms*4,512>>>(a,(float*)dout,n4);},10);
  printf("read 4GiB: %.1f GB/s\n", 1.0*n*4/(ms*1e-3)/1e9);
  CK(cudaDeviceSynchronize());
  return 0;
}
