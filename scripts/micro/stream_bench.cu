// Microbenchmark (not part of the product): streaming 4 SoA columns (u32,u32,f64,f64)
// of N slots through 147 CTAs x 512 threads, (a) cp.async.bulk into a STAGES-deep smem
// ring, (b) 128-bit __ldcg loads, 4 slots per thread; each slot does a trivial reduction.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int NT = 512;
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(b))); }
__device__ __forceinline__ void mb_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(sa(b)), "r"(ph) : "memory"); }
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(d)), "l"(s), "r"(n), "r"(sa(b)) : "memory"); }

template <int TILE, int STAGES, int NTH = NT, bool COMPUTE = true>
__global__ void __launch_bounds__(NTH) k_bulk(const uint32_t* m, const uint32_t* id, const double* l, const double* p, uint64_t N, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  const uint64_t lo = (N * blockIdx.x / gridDim.x) & ~3ull, hi = blockIdx.x + 1 == gridDim.x ? N : ((N * (blockIdx.x + 1) / gridDim.x) & ~3ull);
  const uint64_t nt = (hi - lo + TILE - 1) / TILE;
  constexpr uint32_t TB = TILE * 24;
  auto issue = [&](uint64_t t) {
    int st = t % STAGES; uint64_t t0 = lo + t * TILE; uint32_t n = (uint32_t)min((uint64_t)TILE, hi - t0); n = (n + 3) & ~3u;
    unsigned char* b = sm + st * TB;
    mb_tx(&bar[st], n * 24);
    bulk(b, m + t0, n * 4, &bar[st]); bulk(b + TILE * 4, id + t0, n * 4, &bar[st]);
    bulk(b + TILE * 8, l + t0, n * 8, &bar[st]); bulk(b + TILE * 16, p + t0, n * 8, &bar[st]);
  };
  if (threadIdx.x == 0) { for (int s = 0; s < STAGES; ++s) mb_init(&bar[s]); asm volatile("fence.proxy.async.shared::cta;"); for (uint64_t t = 0; t < nt && t < STAGES; ++t) issue(t); }
  __syncthreads();
  double acc = 0;
  for (uint64_t t = 0; t < nt; ++t) {
    int st = t % STAGES; mb_wait(&bar[st], (t / STAGES) & 1);
    unsigned char* b = sm + st * TB;
    const uint32_t* mm = (const uint32_t*)b; const uint32_t* ii = (const uint32_t*)(b + TILE * 4);
    const double* ll = (const double*)(b + TILE * 8); const double* pp = (const double*)(b + TILE * 16);
    uint64_t t0 = lo + t * TILE; uint32_t n = (uint32_t)min((uint64_t)TILE, hi - t0);
    for (uint32_t k = threadIdx.x; k < n; k += NTH) { if (COMPUTE) { if (mm[k] & 1024) acc += __ddiv_rn(pp[k] * (double)ii[k], 1.0 + ll[k]); } else acc += (double)(mm[k] ^ ii[k]) + ll[k] + pp[k]; }
    __syncthreads();
    if (threadIdx.x == 0 && t + STAGES < nt) issue(t + STAGES);
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void __launch_bounds__(NT, 1) k_ldg(const uint32_t* m, const uint32_t* id, const double* l, const double* p, uint64_t N, double* out) {
  const uint64_t lo = (N * blockIdx.x / gridDim.x) & ~3ull, hi = blockIdx.x + 1 == gridDim.x ? N : ((N * (blockIdx.x + 1) / gridDim.x) & ~3ull);
  double acc = 0;
  for (uint64_t s0 = lo + 4 * threadIdx.x; s0 < hi; s0 += 4 * NT) {
    uint4 mm = __ldcg((const uint4*)(m + s0)); uint4 ii = __ldcg((const uint4*)(id + s0));
    double2 l0 = __ldcg((const double2*)(l + s0)), l1 = __ldcg((const double2*)(l + s0 + 2));
    double2 p0 = __ldcg((const double2*)(p + s0)), p1 = __ldcg((const double2*)(p + s0 + 2));
    if (mm.x & 1024) acc += __ddiv_rn(p0.x * ii.x, 1.0 + l0.x);
    if (mm.y & 1024) acc += __ddiv_rn(p0.y * ii.y, 1.0 + l0.y);
    if (mm.z & 1024) acc += __ddiv_rn(p1.x * ii.z, 1.0 + l1.x);
    if (mm.w & 1024) acc += __ddiv_rn(p1.y * ii.w, 1.0 + l1.y);
  }
  if (acc == 12345.678) out[0] = acc;
}

template <class F> float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a); for (int i = 0; i < 20; ++i) f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms / 20;
}
int main() {
  const uint64_t N = 1ull << 22;
  uint32_t *m, *id; double *l, *p, *out;
  cudaMalloc(&m, N * 4 + 64); cudaMalloc(&id, N * 4 + 64); cudaMalloc(&l, N * 8 + 64); cudaMalloc(&p, N * 8 + 64); cudaMalloc(&out, 8);
  cudaMemset(m, 0xff, N * 4); cudaMemset(id, 1, N * 4); cudaMemset(l, 0, N * 8); cudaMemset(p, 0, N * 8);
  char* flush; cudaMalloc(&flush, 512 << 20);
  int G = 147;
  const double bytes = N * 24.0;
  auto rep = [&](const char* nm, float ms) { printf("%-28s %8.2f us  %7.1f GB/s\n", nm, ms * 1e3, bytes / (ms * 1e-3) / 1e9); };
  float fl = timeit([&] { cudaMemsetAsync(flush, 0, 512 << 20); });
  auto rep2 = [&](const char* nm, float ms) { ms -= fl; printf("%-36s %8.2f us  %7.1f GB/s\n", nm, ms * 1e3, bytes / (ms * 1e-3) / 1e9); };
#define BULK(T, S, NTH, C, GRID) { auto k = k_bulk<T, S, NTH, C>; cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, T * 24 * S); \
   rep2("bulk T" #T " S" #S " nth" #NTH " c" #C " g" #GRID, timeit([&] { cudaMemsetAsync(flush, 0, 512 << 20); k<<<GRID, NTH, T * 24 * S>>>(m, id, l, p, N, out); })); }
  BULK(1024, 4, 512, true, 147) BULK(1024, 8, 512, true, 147) BULK(2048, 4, 512, true, 147) BULK(1024, 6, 512, true, 148) BULK(1024, 4, 512, false, 147) BULK(2048, 4, 512, false, 147) BULK(1024, 8, 512, false, 147)
  BULK(1024, 4, 256, false, 296) BULK(512, 4, 256, false, 592) BULK(2048, 4, 1024, false, 147) BULK(4096, 2, 512, false, 147)
#define BULKNF(T, S, NTH, C, GRID) { auto k = k_bulk<T, S, NTH, C>; cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, T * 24 * S); \
   rep("noflush bulk T" #T " S" #S " nth" #NTH " c" #C " g" #GRID, timeit([&] { k<<<GRID, NTH, T * 24 * S>>>(m, id, l, p, N, out); })); }
  BULKNF(1024, 4, 512, true, 147) BULKNF(1024, 8, 512, true, 147) BULKNF(2048, 4, 512, true, 147) BULKNF(1024, 4, 256, true, 296)
  rep2("ldg 4/thr g147", timeit([&] { cudaMemsetAsync(flush, 0, 512 << 20); k_ldg<<<G, NT>>>(m, id, l, p, N, out); }));
  rep2("ldg 4/thr g592", timeit([&] { cudaMemsetAsync(flush, 0, 512 << 20); k_ldg<<<G * 4, NT>>>(m, id, l, p, N, out); }));
  rep2("ldg 4/thr g2368", timeit([&] { cudaMemsetAsync(flush, 0, 512 << 20); k_ldg<<<G * 16, NT>>>(m, id, l, p, N, out); }));
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
