// workload/csrc/synth.cu -- GPU twin of workload/synth.py (input generator only).
//
// Fabricates the per-stage logits a model cascade would hand the router, keyed
// by (seed, stage, request id, token, class), bit-identical to logits_np().
// Holds none of the method's arithmetic.  Built into workload/libhs_synth.so.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace {

__host__ __device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7FEB352Du; x ^= x >> 15; x *= 0x846CA68Bu; x ^= x >> 16;
  return x;
}
__host__ __device__ __forceinline__ uint32_t seed_key(uint32_t seed) { return mix32(seed ^ 0x5BD1E995u); }
__host__ __device__ __forceinline__ uint32_t id_key(uint32_t base, int64_t id) {
  uint64_t u = (uint64_t)id;
  return mix32(mix32(base ^ (uint32_t)(u & 0xFFFFFFFFu)) ^ (uint32_t)(u >> 32));
}

struct RowInfo { uint32_t tk; int32_t winner; int32_t wcode; };
// winner-code profile (synth.winner_code): rb, rm1, rm2, wb, wm, cs, ccap
struct Margin { int32_t rb, rm1, rm2, wb, wm, cs, ccap; };

__device__ __forceinline__ RowInfo row_info(uint32_t skey, uint32_t stkey, int64_t id, int t, int L,
                                            int64_t C, int64_t thr, const Margin& mg) {
  uint32_t rq = id_key(skey, id);
  uint32_t rk = id_key(stkey, id);
  uint32_t d = mix32(rq ^ 0xD1FFu) & 0xFFFFu;
  uint32_t e = mix32(rk ^ 0xE751u) & 0x7FFFu;
  bool meant = (int64_t)d + (int64_t)e < thr;
  int64_t tstar = (int64_t)(mix32(rk ^ 0x7777u) % (uint32_t)L);
  int64_t lab = (int64_t)(mix32(rq ^ mix32((uint32_t)t + 0x01000193u)) % (uint32_t)C);
  uint32_t tk = mix32(rk + (uint32_t)t * 0x9E3779B9u);
  bool ok = meant || (t != tstar);
  uint32_t cm1 = (uint32_t)(C - 1 > 0 ? C - 1 : 1);
  int64_t other = (int64_t)(mix32(tk ^ 0x0BADu) % cm1);
  int64_t winner = ok ? lab : (lab + 1 + other) % C;
  int64_t m1 = mix32(tk ^ 0x11u), m2 = mix32(tk ^ 0x22u);
  int64_t right = mg.rb + (m1 & mg.rm1) + (m2 & mg.rm2);
  if (mg.cs > 0) {
    int64_t slack = thr - (int64_t)d - (int64_t)e;
    slack = slack > 0 ? slack >> mg.cs : 0;
    right += slack < mg.ccap ? slack : mg.ccap;
  }
  int32_t wcode = ok ? (int32_t)right : (int32_t)(mg.wb + (m1 & mg.wm));
  RowInfo r; r.tk = tk; r.winner = (int32_t)winner; r.wcode = wcode;
  return r;
}

__device__ __forceinline__ int32_t bg_code(uint32_t tk, int64_t j) {
  uint32_t h = mix32(tk + (uint32_t)(j + 1) * 0x85EBCA6Bu);
  int32_t s = (int32_t)((h & 255u) + ((h >> 8) & 255u) + ((h >> 16) & 255u) + (h >> 24));
  return (s - 510) >> 3;
}

// One CTA-stripe per logits row (n*L rows), threads over classes.
template <bool BF16>
__global__ void synth_logits_kernel(void* out, const int64_t* ids, int64_t id_base, int64_t n, int L,
                                    int64_t C, int64_t stride, uint32_t skey, uint32_t stkey,
                                    int64_t thr, float scale, Margin mg) {
  for (int64_t row = blockIdx.x; row < n * L; row += gridDim.x) {
    int64_t i = row / L;
    int t = (int)(row % L);
    int64_t id = ids ? ids[i] : id_base + i;
    RowInfo ri = row_info(skey, stkey, id, t, L, C, thr, mg);
    for (int64_t j = threadIdx.x; j < C; j += blockDim.x) {
      int32_t code = (j == ri.winner) ? ri.wcode : bg_code(ri.tk, j);
      float v = (float)code * scale;
      if (BF16) {
        uint32_t u = __float_as_uint(v);           // exact: <= 8 significant bits
        ((uint16_t*)out)[row * stride + j] = (uint16_t)(u >> 16);
      } else {
        ((float*)out)[row * stride + j] = v;
      }
    }
  }
}

__global__ void synth_labels_kernel(int32_t* out, const int64_t* ids, int64_t id_base, int64_t n,
                                    int L, int64_t C, uint32_t skey) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n * L) return;
  int64_t i = k / L;
  int t = (int)(k % L);
  int64_t id = ids ? ids[i] : id_base + i;
  uint32_t rq = id_key(skey, id);
  out[k] = (int32_t)(mix32(rq ^ mix32((uint32_t)t + 0x01000193u)) % (uint32_t)C);
}

}  // namespace

extern "C" {

// out: device [n*L rows x stride]; ids: device int64[n] or NULL (ids = id_base + i).
// dtype: 0 fp32, 1 bf16.  margin: host int32[7] (synth.winner_code).
// Returns a cudaError_t value (0 = success).
int hs_synth_logits(void* out, int dtype, const int64_t* ids, int64_t id_base, int64_t n, int L,
                    int64_t C, int64_t stride, int stage, uint32_t seed, int64_t thr,
                    int scale_log2, const int32_t* margin, cudaStream_t s) {
  if (n <= 0) return 0;
  Margin mg = {margin[0], margin[1], margin[2], margin[3], margin[4], margin[5], margin[6]};
  uint32_t skey = seed_key(seed);
  uint32_t stkey = mix32(skey ^ mix32((uint32_t)stage + 0x27D4EB2Fu));
  float scale = ldexpf(1.0f, -scale_log2);
  int64_t rows = n * L;
  int grid = (int)(rows < (1 << 20) ? rows : (1 << 20));
  int block = C >= 1024 ? 512 : 256;
  if (dtype == 1)
    synth_logits_kernel<true><<<grid, block, 0, s>>>(out, ids, id_base, n, L, C, stride, skey, stkey, thr, scale, mg);
  else
    synth_logits_kernel<false><<<grid, block, 0, s>>>(out, ids, id_base, n, L, C, stride, skey, stkey, thr, scale, mg);
  return (int)cudaGetLastError();
}

int hs_synth_labels(int32_t* out, const int64_t* ids, int64_t id_base, int64_t n, int L, int64_t C,
                    uint32_t seed, cudaStream_t s) {
  if (n <= 0) return 0;
  int64_t tot = n * L;
  synth_labels_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(out, ids, id_base, n, L, C, seed_key(seed));
  return (int)cudaGetLastError();
}

}  // extern "C"
