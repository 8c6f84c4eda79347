// Multi-turn session predictor (Eq.(4)) on the sm_100a tensor cores.
//
//   y = W3 relu(W2 relu(W1 h + b1) + b2) + b3,   prediction = (y > 0)      (A43-A45)
//
// h: the serving model's final-layer hidden state of the request's last prompt token
// (bf16, d wide), W1: 256 x d, W2: 64 x 256 (bf16), b1, b2, W3 (1 x 64), b3 in fp32.
//
// One persistent CTA per SM walks 256-row tiles of H.  Per tile:
//   GEMM1  D1[mt] (128 x 256 fp32, TMEM columns mt*256..) = H[mt rows] . W1^T  for mt = 0, 1:
//          both M tiles consume every W1 k-block once (halves the W1 traffic from L2);
//          operands arrive by TMA (SWIZZLE_64B, 32-wide k-blocks, 4-stage ring), one elected
//          thread issues tcgen05.mma (kind::f16, M=128, N=256, K=16), tcgen05.commit frees a
//          stage back to the TMA warp.
//   EPI1   4 epilogue warps (one TMEM lane = one row per thread) read D1 with tcgen05.ld,
//          add b1, ReLU, round to bf16 and write the GEMM2 A operand to shared memory in the
//          SWIZZLE_128B K-major layout.
//   GEMM2  D2 (128 x 64 fp32, in the drained D1 columns) = relu1 . W2^T (W2 resident in smem).
//   EPI2   tcgen05.ld D2, add b2, ReLU, dot W3 in fp32 (index order), add b3 -> logit; the
//          prediction bit goes to the request's flags byte (b0 = is_multi_turn, sae_batch).
// Roles: warp 0 TMA producer, warp 1 TMEM owner + MMA issuer, warps 2-5 epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "sae.h"

namespace pred {

constexpr int BM = 128;                       // rows per M tile (TMEM lanes)
constexpr int MT = 2;                         // M tiles per CTA tile
constexpr int ROWS = BM * MT;                 // 256 rows per CTA tile
constexpr int N1 = 256, N2 = 64;              // hidden widths
constexpr int BK = 32;                        // k-block: 32 bf16 = one 64 B swizzle row
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;          // 8 KB
constexpr int B_BYTES = N1 * BK * 2;          // 16 KB
constexpr int STAGE_BYTES = MT * A_BYTES + B_BYTES;   // 32 KB
constexpr int H1_BYTES = BM * N1 * 2;         // 64 KB: 4 k-atoms x 128 rows x 128 B
constexpr int W2_BYTES = N2 * N1 * 2;         // 32 KB: 4 k-atoms x 64 rows x 128 B
constexpr int OFF_H1 = STAGES * STAGE_BYTES;
constexpr int OFF_W2 = OFF_H1 + H1_BYTES;
constexpr int OFF_MISC = OFF_W2 + W2_BYTES;
// misc: 8 B barriers, tmem base, biases
constexpr int NBAR = 2 * STAGES + 5;
constexpr int OFF_BAR = OFF_MISC;
constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
constexpr int OFF_B1 = OFF_TMEM + 16;
constexpr int OFF_B2 = OFF_B1 + N1 * 4;
constexpr int OFF_W3 = OFF_B2 + N2 * 4;
constexpr int OFF_B3 = OFF_W3 + N2 * 4;
constexpr int SMEM_USED = OFF_B3 + 16;
constexpr int SMEM_TOTAL = SMEM_USED + 1024;  // + alignment slack of the dynamic base
constexpr int NTHREADS = 192;
constexpr uint32_t TMEM_COLS = 512;

// instruction descriptors (kind::f16): D f32 (bit 4), A/B bf16 (bits 7, 10), K-major A/B,
// N >> 3 at bit 17, M >> 4 at bit 24
constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
constexpr uint32_t IDESC1 = idesc(128, N1);
constexpr uint32_t IDESC2 = idesc(128, N2);

// shared-memory matrix descriptor, K-major, swizzled: start >> 4, LBO (unused) 1,
// SBO = 8 rows x row bytes, version 1 (sm100), layout type (2 = 128B, 4 = 64B)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) |
         ((uint64_t)1u << 46) | ((uint64_t)layout << 61);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(b),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* tm, int x, int y, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"((uint64_t)tm), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mma_f16(uint32_t dtmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(dtmem),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

struct Args {
  uint32_t n;            // rows of H
  uint32_t nkb;          // d / BK
  const float* b1;       // [256]
  const float* b2;       // [64]
  const float* w3;       // [64]
  float b3;
  const uint32_t* rows;  // optional: output index of prediction i
  float* logit;          // optional [n]
  uint8_t* flags;        // optional: b0 := prediction
};

__global__ void __launch_bounds__(NTHREADS, 1)
    k_predict(const __grid_constant__ CUtensorMap tm_h, const __grid_constant__ CUtensorMap tm_w1,
              const __grid_constant__ CUtensorMap tm_w2, Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = smem_u32(sm);
  const uint32_t bar0 = sbase + OFF_BAR;
  auto full = [&](int s) { return bar0 + 8u * s; };
  auto empty = [&](int s) { return bar0 + 8u * (STAGES + s); };
  const uint32_t accum_full = bar0 + 8u * (2 * STAGES);
  const uint32_t h1_full = accum_full + 8, d2_full = accum_full + 16, tmem_empty = accum_full + 24,
                 w2_full = accum_full + 32;
  uint32_t* tmem_slot = (uint32_t*)(sm + OFF_TMEM);
  float* sb1 = (float*)(sm + OFF_B1);
  float* sb2 = (float*)(sm + OFF_B2);
  float* sw3 = (float*)(sm + OFF_W3);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ntiles = (a.n + ROWS - 1) / ROWS;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(full(s), 1); mbar_init(empty(s), 1); }
    mbar_init(accum_full, 1);
    mbar_init(h1_full, 1);
    mbar_init(d2_full, 1);
    mbar_init(tmem_empty, 1);
    mbar_init(w2_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tm_h) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tm_w1) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp >= 2) {
    const int t = threadIdx.x - 64;
    for (int i = t; i < N1; i += 128) sb1[i] = a.b1[i];
    if (t < N2) { sb2[t] = a.b2[t]; sw3[t] = a.w3[t]; }
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      mbar_expect_tx(w2_full, W2_BYTES);
      for (int k = 0; k < 4; ++k) tma_load_2d(sbase + OFF_W2 + k * 8192, &tm_w2, k * 64, 0, w2_full);
      uint32_t s = 0, ph = 0;
      for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int row0 = (int)(tile * ROWS);
        for (uint32_t kb = 0; kb < a.nkb; ++kb) {
          mbar_wait(empty(s), ph ^ 1u);
          const uint32_t st = sbase + s * STAGE_BYTES;
          mbar_expect_tx(full(s), STAGE_BYTES);
          tma_load_2d(st, &tm_h, (int)(kb * BK), row0, full(s));
          tma_load_2d(st + A_BYTES, &tm_h, (int)(kb * BK), row0 + BM, full(s));
          tma_load_2d(st + MT * A_BYTES, &tm_w1, (int)(kb * BK), 0, full(s));
          if (++s == STAGES) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (one thread) =====
    uint32_t s = 0, ph = 0, it = 0;
    mbar_wait(w2_full, 0);
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      if (it > 0) {
        mbar_wait(tmem_empty, (it - 1) & 1u);
        fence_after();
      }
      for (uint32_t kb = 0; kb < a.nkb; ++kb) {
        mbar_wait(full(s), ph);
        fence_after();
        if (lane == 0) {
          const uint32_t st = sbase + s * STAGE_BYTES;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int ks = 0; ks < BK / 16; ++ks)
              mma_f16(tmem + mt * N1, sdesc(st + mt * A_BYTES + ks * 32, 512, 4),
                      sdesc(st + MT * A_BYTES + ks * 32, 512, 4), IDESC1, (kb | ks) != 0);
          mma_commit(empty(s));
        }
        __syncwarp();
        if (++s == STAGES) { s = 0; ph ^= 1u; }
      }
      if (lane == 0) mma_commit(accum_full);
      __syncwarp();
      for (int mt = 0; mt < MT; ++mt) {
        mbar_wait(h1_full, (uint32_t)mt & 1u);
        fence_after();
        if (lane == 0) {
#pragma unroll
          for (int ks = 0; ks < N1 / 16; ++ks) {
            const uint32_t at = ks >> 2, ko = (ks & 3) * 32;
            mma_f16(tmem + mt * N1, sdesc(sbase + OFF_H1 + at * 16384 + ko, 1024, 2),
                    sdesc(sbase + OFF_W2 + at * 8192 + ko, 1024, 2), IDESC2, ks != 0);
          }
          mma_commit(d2_full);
        }
        __syncwarp();
      }
    }
  } else {
    // ===== epilogue: warps 2..5, TMEM lane quadrant warp % 4, one row per thread =====
    const uint32_t q = (uint32_t)(warp & 3);
    const uint32_t r = q * 32 + lane;                 // row within the M tile
    const uint32_t lane_addr = (q * 32) << 16;
    uint8_t* h1 = sm + OFF_H1;
    const float b3 = a.b3;
    uint32_t it = 0;
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      mbar_wait(accum_full, it & 1u);
      fence_after();
      for (int mt = 0; mt < MT; ++mt) {
        // EPI1: relu(D1 + b1) -> bf16, SWIZZLE_128B K-major (k-atom of 64 columns = 16 KB)
        for (int ch = 0; ch < N1 / 32; ++ch) {
          float v[32];
          tmem_ld32(tmem + lane_addr + mt * N1 + ch * 32, v);
          uint32_t w[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float x0 = fmaxf(__fadd_rn(v[2 * i], sb1[ch * 32 + 2 * i]), 0.0f);
            const float x1 = fmaxf(__fadd_rn(v[2 * i + 1], sb1[ch * 32 + 2 * i + 1]), 0.0f);
            const __nv_bfloat162 p = __floats2bfloat162_rn(x0, x1);
            w[i] = *reinterpret_cast<const uint32_t*>(&p);
          }
          const uint32_t atom = (uint32_t)ch >> 1, ub = ((uint32_t)ch & 1u) * 4u;
          uint8_t* rowp = h1 + atom * 16384 + r * 128;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t pu = (ub + u) ^ (r & 7u);
            *reinterpret_cast<uint4*>(rowp + pu * 16) = make_uint4(w[4 * u], w[4 * u + 1], w[4 * u + 2], w[4 * u + 3]);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        fence_before();
        epi_sync();
        if (threadIdx.x == 64) mbar_arrive(h1_full);
        // EPI2: relu(D2 + b2) . W3 + b3
        mbar_wait(d2_full, (uint32_t)mt & 1u);
        fence_after();
        float y = 0.0f;
        for (int ch = 0; ch < N2 / 32; ++ch) {
          float v[32];
          tmem_ld32(tmem + lane_addr + mt * N1 + ch * 32, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float x = fmaxf(__fadd_rn(v[i], sb2[ch * 32 + i]), 0.0f);
            y = __fadd_rn(y, __fmul_rn(sw3[ch * 32 + i], x));
          }
        }
        y = __fadd_rn(y, b3);
        const uint32_t row = tile * ROWS + mt * BM + r;
        if (row < a.n) {
          const uint32_t o = a.rows ? a.rows[row] : row;
          if (a.logit) a.logit[o] = y;
          if (a.flags) a.flags[o] = (uint8_t)((a.flags[o] & 0xFEu) | (y > 0.0f ? 1u : 0u));
        }
      }
      fence_before();
      epi_sync();
      if (threadIdx.x == 64) mbar_arrive(tmem_empty);
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
}

}  // namespace pred

// ===========================================================================
// Host side: C ABI (include/sae.h, "Session predictor")
// ===========================================================================
struct sae_predictor {
  int device = 0;
  uint32_t d = 0;
  int nsm = 0;
  void* w1 = nullptr;   // bf16 [256 x d]
  void* w2 = nullptr;   // bf16 [64 x 256]
  float* bias = nullptr;  // b1[256] | b2[64] | w3[64]
  float b3 = 0.0f;
  CUtensorMap tm_w1, tm_w2;
  uint64_t launches = 0;
  std::string err;
};

static std::string g_pred_err;
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}
// 2-D bf16 row-major [rows x cols] tensor map with a (box_cols x box_rows) box
static bool make_map(CUtensorMap* tm, const void* base, uint64_t rows, uint64_t cols, uint32_t box_cols,
                     uint32_t box_rows, CUtensorMapSwizzle sw) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

extern "C" {

sae_status sae_predictor_create(const sae_predictor_config* cfg, const uint16_t* w1, const float* b1,
                                const uint16_t* w2, const float* b2, const float* w3, float b3,
                                sae_predictor** out) {
  if (!cfg || !w1 || !b1 || !w2 || !b2 || !w3 || !out) { g_pred_err = "null argument"; return SAE_E_INVAL; }
  if (cfg->abi_version != SAE_ABI_VERSION) { g_pred_err = "ABI version mismatch"; return SAE_E_ABI; }
  if (cfg->d == 0 || cfg->d % pred::BK != 0 || cfg->d > (1u << 20)) {
    g_pred_err = "hidden size d must be a positive multiple of 32";
    return SAE_E_INVAL;
  }
  if (cudaSetDevice(cfg->device) != cudaSuccess) { g_pred_err = "cudaSetDevice failed"; return SAE_E_CUDA; }
  sae_predictor* p = new sae_predictor();
  p->device = cfg->device;
  p->d = cfg->d;
  p->b3 = b3;
  auto fail = [&](sae_status st, const char* why) {
    cudaFree(p->w1); cudaFree(p->w2); cudaFree(p->bias);
    delete p;
    g_pred_err = why;
    return st;
  };
  const size_t w1b = (size_t)pred::N1 * cfg->d * 2, w2b = (size_t)pred::N2 * pred::N1 * 2;
  if (cudaMalloc(&p->w1, w1b) != cudaSuccess || cudaMalloc(&p->w2, w2b) != cudaSuccess ||
      cudaMalloc(&p->bias, (pred::N1 + 2 * pred::N2) * sizeof(float)) != cudaSuccess)
    return fail(SAE_E_OOM, "cudaMalloc failed");
  if (cudaMemcpy(p->w1, w1, w1b, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->w2, w2, w2b, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->bias, b1, pred::N1 * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->bias + pred::N1, b2, pred::N2 * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->bias + pred::N1 + pred::N2, w3, pred::N2 * 4, cudaMemcpyHostToDevice) != cudaSuccess)
    return fail(SAE_E_CUDA, "cudaMemcpy failed");
  if (!make_map(&p->tm_w1, p->w1, pred::N1, cfg->d, pred::BK, pred::N1, CU_TENSOR_MAP_SWIZZLE_64B) ||
      !make_map(&p->tm_w2, p->w2, pred::N2, pred::N1, 64, pred::N2, CU_TENSOR_MAP_SWIZZLE_128B))
    return fail(SAE_E_CUDA, "cuTensorMapEncodeTiled failed (weights)");
  if (cudaDeviceGetAttribute(&p->nsm, cudaDevAttrMultiProcessorCount, cfg->device) != cudaSuccess ||
      cudaFuncSetAttribute(pred::k_predict, cudaFuncAttributeMaxDynamicSharedMemorySize, pred::SMEM_TOTAL) !=
          cudaSuccess)
    return fail(SAE_E_CUDA, "device attribute / smem opt-in failed");
  *out = p;
  return SAE_OK;
}

sae_status sae_predictor_destroy(sae_predictor* p) {
  if (!p) return SAE_E_INVAL;
  cudaSetDevice(p->device);
  cudaDeviceSynchronize();
  cudaFree(p->w1); cudaFree(p->w2); cudaFree(p->bias);
  delete p;
  return SAE_OK;
}

sae_status sae_predict(sae_predictor* p, const uint16_t* h, uint32_t n, const uint32_t* rows, float* logit,
                       uint8_t* flags, sae_stream s) {
  if (!p) { g_pred_err = "null predictor"; return SAE_E_INVAL; }
  if (n == 0) return SAE_OK;
  if (!h || (!logit && !flags)) { p->err = "null input or no output"; return SAE_E_INVAL; }
  if (((uintptr_t)h & 15u) != 0) { p->err = "hidden states must be 16-byte aligned"; return SAE_E_INVAL; }
  CUtensorMap tm_h;
  if (!make_map(&tm_h, h, n, p->d, pred::BK, pred::BM, CU_TENSOR_MAP_SWIZZLE_64B)) {
    p->err = "cuTensorMapEncodeTiled failed (hidden states)";
    return SAE_E_CUDA;
  }
  pred::Args a;
  a.n = n;
  a.nkb = p->d / pred::BK;
  a.b1 = p->bias;
  a.b2 = p->bias + pred::N1;
  a.w3 = p->bias + pred::N1 + pred::N2;
  a.b3 = p->b3;
  a.rows = rows;
  a.logit = logit;
  a.flags = flags;
  const uint32_t ntiles = (n + pred::ROWS - 1) / pred::ROWS;
  const uint32_t grid = ntiles < (uint32_t)p->nsm ? ntiles : (uint32_t)p->nsm;
  pred::k_predict<<<grid, pred::NTHREADS, pred::SMEM_TOTAL, (cudaStream_t)s>>>(tm_h, p->tm_w1, p->tm_w2, a);
  p->launches++;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { p->err = cudaGetErrorString(e); return SAE_E_CUDA; }
  return SAE_OK;
}

uint64_t sae_predictor_launch_count(const sae_predictor* p) { return p ? p->launches : 0; }

const char* sae_predictor_last_error(const sae_predictor* p) {
  return p ? p->err.c_str() : g_pred_err.c_str();
}

}  // extern "C"
