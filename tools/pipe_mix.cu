// Microbenchmark: which pipe the K2 softmax's instructions share.  Per thread 16 independent
// fp32 lanes; each mode issues a fixed instruction mix per iteration; cycles per iteration per
// SM are reported so that mixes can be compared with the sum of their parts (same pipe) or the
// max (different pipes).
//   ex2      16 x MUFU.EX2 (ex2.approx.ftz.f32)
//   cvt      8 x F2FP bf16x2 pack (cvt.rn.bf16x2.f32)
//   ex2+cvt  both
//   ex2bf    8 x ex2.approx.ftz.bf16x2 (two exps per lane per instruction, packed bf16 out)
//   ipack    8 x integer bf16 pack (two IADD + one PRMT: round-half-up on the upper 16 bits)
//   ex2+ipk  16 x MUFU.EX2 + 8 integer packs
//   ffma2    8 x FFMA2
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t cvt2(float lo, float hi) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint32_t ex2bf(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t ipack(float lo, float hi) {
  const uint32_t a = __float_as_uint(lo) + 0x8000u, b = __float_as_uint(hi) + 0x8000u;
  uint32_t r;
  asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

template <int MODE>
__global__ void __launch_bounds__(256) k(float* out, int iters, long long* cyc) {
  float v[16];
  uint32_t u[8];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = -0.001f * (threadIdx.x + i);
#pragma unroll
  for (int i = 0; i < 8; ++i) u[i] = 0x3f803f80u + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0 || MODE == 2 || MODE == 5) {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = ex2f(v[i]) - 1.0f;
    }
    if (MODE == 1 || MODE == 2) {
#pragma unroll
      for (int i = 0; i < 8; ++i) u[i] ^= cvt2(v[2 * i] + u[i], v[2 * i + 1]);
    }
    if (MODE == 3) {
#pragma unroll
      for (int i = 0; i < 8; ++i) u[i] = ex2bf(u[i]) ^ 0x80008000u;
    }
    if (MODE == 4 || MODE == 5) {
#pragma unroll
      for (int i = 0; i < 8; ++i) u[i] ^= ipack(v[2 * i] + u[i], v[2 * i + 1]);
    }
    if (MODE == 6) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float2 a = make_float2(v[2 * i], v[2 * i + 1]);
        a = __ffma2_rn(a, make_float2(0.999f, 0.998f), make_float2(0.001f, 0.002f));
        v[2 * i] = a.x;
        v[2 * i + 1] = a.y;
      }
    }
    if (MODE >= 7 && MODE <= 11) {
      // the K2 exp loop's per-pair mix: FFMA2 (scale), 2 x MUFU.EX2, FADD2 (row sum), F2FP (pack)
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float2 x = make_float2(v[2 * i], v[2 * i + 1]);
        if (MODE != 10) x = __ffma2_rn(x, make_float2(1.0001f, 1.0001f), make_float2(-0.5f, -0.5f));
        float2 p = x;
        if (MODE == 7 || MODE == 8) { p.x = ex2f(x.x); p.y = ex2f(x.y); }
        if (MODE != 11) acc = __fadd2_rn(acc, p);
        if (MODE == 7 || MODE == 9 || MODE == 11) u[i] ^= cvt2(p.x, p.y);
        v[2 * i] = p.x - 0.25f;
        v[2 * i + 1] = p.y - 0.25f;
      }
      v[0] += acc.x;
      v[1] += acc.y;
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += v[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += __uint_as_float(u[i]);
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int MODE>
void run(const char* name, int threads) {
  float* o;
  long long* c;
  cudaMalloc(&o, 4);
  cudaMalloc(&c, 8);
  const int iters = 4000;
  k<MODE><<<148, threads>>>(o, 10, c);
  cudaDeviceSynchronize();
  k<MODE><<<148, threads>>>(o, iters, c);
  cudaDeviceSynchronize();
  long long cyc;
  cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
  // cycles one SM spends per iteration of one warp's worth of threads, per warp
  printf("%-8s threads=%3d: %7.1f cycles per warp-iteration per SMSP\n", name, threads,
         double(cyc) / iters / (threads / 32 / 4.0));
}

int main() {
  for (int t : {128, 256}) {
    run<0>("ex2", t);
    run<1>("cvt", t);
    run<2>("ex2+cvt", t);
    run<3>("ex2bf", t);
    run<4>("ipack", t);
    run<5>("ex2+ipk", t);
    run<6>("ffma2", t);
    run<7>("pair-all", t);
    run<8>("pair-nocvt", t);
    run<9>("pair-nomufu", t);
    run<10>("fadd2+cvt", t);
    run<11>("ffma2+cvt", t);
  }
  return 0;
}
