// aux.cu -- small helper kernels around the attention launch:
//   * pack the u8 key mask (Evoformer MSA mask, G9) into one bit per key so the
//     attention kernels test a key with a shift instead of a strided byte load;
//   * write the S_k == 0 / no-work result (O = 0, lse = -inf, reading G7).
#include <cuda_runtime.h>
#include <math.h>

#include "params.h"

namespace fl {

// keybits[(b*G + g) * words + w] bit t = key_mask[b, g, 32*w + t] != 0 (0 beyond S_k).
__global__ void pack_keymask_kernel(const unsigned char* km, int64_t sb, int64_t sg, int64_t sk, int B, int G, int Sk,
                                    int words, uint32_t* out) {
  const int64_t total = (int64_t)B * G * words;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int w = (int)(i % words);
    const int64_t bg = i / words;
    const int g = (int)(bg % G), b = (int)(bg / G);
    uint32_t bits = 0;
    for (int t = 0; t < 32; ++t) {
      const int k = w * 32 + t;
      if (k < Sk && km[b * sb + g * sg + (int64_t)k * sk] != 0) bits |= 1u << t;
    }
    out[i] = bits;
  }
}

cudaError_t launch_pack_keymask(const unsigned char* km, int64_t sb, int64_t sg, int64_t sk, int B, int G, int Sk,
                                int words, uint32_t* out, cudaStream_t stream) {
  const int64_t total = (int64_t)B * G * words;
  const int threads = 256;
  const int blocks = (int)((total + threads - 1) / threads < 148 * 8 ? (total + threads - 1) / threads : 148 * 8);
  pack_keymask_kernel<<<blocks > 0 ? blocks : 1, threads, 0, stream>>>(km, sb, sg, sk, B, G, Sk, words, out);
  return cudaGetLastError();
}

// O = 0 (bf16 or f32, strided [B,G,H,S,D]) and lse = -inf for every row.
__global__ void fill_empty_kernel(AttnParams p) {
  const int64_t rows = (int64_t)p.B * p.G * p.Hq * p.Sq;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * p.Dv;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int d = (int)(i % p.Dv);
    int64_t r = i / p.Dv;
    const int q = (int)(r % p.Sq);
    r /= p.Sq;
    const int h = (int)(r % p.Hq);
    r /= p.Hq;
    const int g = (int)(r % p.G), b = (int)(r / p.G);
    const int64_t off = b * p.os.b + g * p.os.g + h * p.os.h + (int64_t)q * p.os.s + d;
    if (p.in_dtype == 1)
      static_cast<float*>(p.o)[off] = 0.f;
    else
      static_cast<unsigned short*>(p.o)[off] = 0;
    if (d == 0 && p.lse) p.lse[b * p.lses.b + g * p.lses.g + h * p.lses.h + (int64_t)q * p.lses.s] = -INFINITY;
  }
}

cudaError_t launch_fill_empty(const AttnParams& p, cudaStream_t stream) {
  const int64_t n = (int64_t)p.B * p.G * p.Hq * p.Sq * p.Dv;
  const int threads = 256;
  int64_t blocks = (n + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  fill_empty_kernel<<<(unsigned)(blocks > 0 ? blocks : 1), threads, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace fl
