// host.cu -- the C ABI of include/fl_attn.h: validation, descriptor -> device
// params, TMA tensor-map encoding, kernel selection and launch.  No device
// memory is ever allocated here and nothing synchronises; there is no fallback:
// anything the kernels do not implement returns FL_ERR_UNSUPPORTED.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <initializer_list>
#include <mutex>
#include <string>

#include "../../include/fl_attn.h"
#include "params.h"

namespace fl {
cudaError_t launch_attn_simt(const AttnParams& p, cudaStream_t stream);
cudaError_t launch_attn_tc(const AttnParams& p, const TmaMaps& maps, cudaStream_t stream);
cudaError_t launch_ipa_prep(const IpaParams& p, cudaStream_t s);
cudaError_t launch_ipa_finish(const IpaParams& p, const float* lse, float* A, void* opair, float* op, cudaStream_t s);
size_t ipa_out_smem(const IpaParams& p);
int linear_nt_max();
cudaError_t launch_linear(const LinParams& p, const CUtensorMap& tx, const CUtensorMap& tw, const CUtensorMap& ty,
                          int y_tma, cudaStream_t stream);
cudaError_t launch_pack_keymask(const unsigned char* km, int64_t sb, int64_t sg, int64_t sk, int B, int G, int Sk,
                                int words, uint32_t* out, cudaStream_t stream);
cudaError_t launch_fill_empty(const AttnParams& p, cudaStream_t stream);
cudaError_t launch_diag_gemm(int n, int k, const CUtensorMap& ta, const CUtensorMap& tb, const void* a, float* c,
                             bool bmn, bool atmem, cudaStream_t s);
int tc_chunk_elems(int D);
cudaError_t launch_rsa_summaries(const void* k, int64_t sb, int64_t sg, int64_t sh, int64_t ss, int B, int G, int H,
                                 int Sk, int D, int blk, int j0, void* kmin, void* kmax, cudaStream_t stream);
cudaError_t launch_rsa_select(const RsaSelParams& p, const CUtensorMap& tq, const CUtensorMap& tmin,
                              const CUtensorMap& tmax, cudaStream_t stream);
int rsa_select_max_blocks(int D);
bool rsa_select_small_ok(const RsaSelParams& p);
cudaError_t launch_rsa_select_small(const RsaSelParams& p, const void* q, int64_t qsb, int64_t qsg, int64_t qsh,
                                    int64_t qss, const void* kmin, const void* kmax, cudaStream_t stream);
size_t decode_workspace_bytes(const AttnParams& p, int n_sms);
cudaError_t launch_attn_decode(const AttnParams& p, const TmaMaps& maps, float* part, int n_sms, cudaStream_t stream);
cudaError_t debug_timing(unsigned long long* out, int reset);
cudaError_t launch_pipe_rate(int op, int iters, int n_sms, float* sink, cudaStream_t s);
cudaError_t launch_sched_dump(const AttnParams& p, int32_t* out, int64_t out_words, int64_t* n_records,
                              int32_t* max_tiles, cudaStream_t stream);
cudaError_t launch_bwd_prepass(const AttnParams& p, const void* dout, Strided5 dos, float* dvec, void* da, void* dgate,
                               Strided5 dgs, const void* aun, cudaStream_t s);
cudaError_t launch_zero_rows(void* dst, Strided5 ds, int B, int G, int H, int S, int D, cudaStream_t s);
cudaError_t launch_diff_bwd_seed(const AttnParams& p, const void* dout, Strided5 dos, const void* o1, void* do1,
                                 float* dlambda, cudaStream_t s);
cudaError_t launch_attn_bwd(const AttnParams& p, const TmaMaps& maps, const CUtensorMap& tdo, const CUtensorMap& tq64,
                            const CUtensorMap& tdo64, const float* lse,
                            Strided5 ls, const void* dout, Strided5 dos, float* dvec, void* dq, Strided5 dqs, void* dk,
                            Strided5 dks, void* dv, Strided5 dvs, float* dbias, Strided5 dbs, cudaStream_t s);
}  // namespace fl

using namespace fl;

namespace {

constexpr size_t kSchedBytes = 256;   // persistent-scheduler counter region at the head of the workspace

int device_sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    cudaGetLastError();
    return 148;
  }
  if (!cache[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) cudaGetLastError();
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

thread_local std::string g_err;
thread_local int64_t g_launches = 0;

fl_status fail(fl_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

fl_status cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();                     // a failed launch / attribute call must not leak into the next call
  return fail(FL_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

// ---------------------------------------------------------------- driver entry point
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;
std::once_flag g_encode_once;

EncodeTiledFn encode_fn() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<EncodeTiledFn>(fn);
  });
  return g_encode;
}

// ---------------------------------------------------------------- tensor views
// Every tensor is normalised to a 5-D view [B, G, H, S, X]; rank-(4-r) inputs
// get G = 1.  X is D for q/k/v/o/gate, S_k for bias, 1 for lse.
struct View5 {
  bool present = false;
  void* data = nullptr;
  int dtype = 0;
  int64_t size[5] = {1, 1, 1, 1, 1};
  int64_t stride[5] = {0, 0, 0, 0, 0};
};

int elem_bytes(int dtype) { return dtype == FL_F32 || dtype == FL_I32 ? 4 : dtype == FL_U8 ? 1 : 2; }

// Map a rank-(base) or rank-(base+1) tensor onto slots; `slots` lists the View5
// slot of each dim of the rank-(base+1) form (the G dim is slot 1).
// A tensor argument is given when it has data, or when it has no elements (torch hands out NULL for those).
bool given(const fl_tensor& t) {
  if (t.data) return true;
  if (t.rank <= 0 || t.rank > 5) return false;
  for (int d = 0; d < t.rank; ++d)
    if (t.size[d] == 0) return true;
  return false;
}

bool to_view(const fl_tensor& t, int q_rank, int rank_delta, View5& v) {
  v = View5();
  if (!given(t)) return true;                 // absent (an empty tensor with NULL data is present, 0 elements)
  if (t.rank != q_rank + rank_delta) return false;
  v.present = true;
  v.data = t.data;
  v.dtype = t.dtype;
  // full 5-slot order is B,G,H,S,X; rank_delta removes trailing slots (lse: X; key_mask: H... handled by caller)
  const int n5 = 5 + rank_delta;              // number of slots used in the rank-5 (with G) form
  int slot[5];
  if (q_rank == 5) {
    for (int i = 0; i < n5; ++i) slot[i] = i;
  } else {
    slot[0] = 0;
    for (int i = 1; i < t.rank; ++i) slot[i] = i + 1;
  }
  for (int i = 0; i < t.rank; ++i) {
    if (t.size[i] < 0) return false;
    v.size[slot[i]] = t.size[i];
    v.stride[slot[i]] = t.stride[i];
  }
  return true;
}

void byte_range(const View5& v, uintptr_t& lo, uintptr_t& hi) {
  int64_t mn = 0, mx = 0;
  for (int i = 0; i < 5; ++i) {
    if (v.size[i] == 0) {
      lo = hi = 0;
      return;
    }
    const int64_t e = (v.size[i] - 1) * v.stride[i];
    if (e < 0) mn += e; else mx += e;
  }
  const int eb = elem_bytes(v.dtype);
  lo = reinterpret_cast<uintptr_t>(v.data) + mn * eb;
  hi = reinterpret_cast<uintptr_t>(v.data) + (mx + 1) * eb;
}

bool overlaps(const View5& a, const View5& b) {
  if (!a.present || !b.present) return false;
  uintptr_t al, ah, bl, bh;
  byte_range(a, al, ah);
  byte_range(b, bl, bh);
  return al < bh && bl < ah;
}

Strided5 strides_of(const View5& v) {
  return Strided5{v.size[0] > 1 ? v.stride[0] : 0, v.size[1] > 1 ? v.stride[1] : 0, v.size[2] > 1 ? v.stride[2] : 0,
                  v.size[3] > 1 ? v.stride[3] : 0, v.size[4] > 1 ? v.stride[4] : 1};
}

bool on_device(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

bool aligned16(const View5& v) {
  if (reinterpret_cast<uintptr_t>(v.data) % 16) return false;
  for (int i = 0; i < 4; ++i)
    if (v.size[i] > 1 && (v.stride[i] * elem_bytes(v.dtype)) % 16) return false;
  return true;
}

// Encode a 5-D bf16 tensor map (D, S, H, G, B) with box {CH, 128, 1, 1, 1}.
fl_status encode_map(const View5& v, int ch, CUtensorMap* out, int* bcast_g, int* bcast_b, int box_rows = 128) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(FL_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable (driver too old?)");
  cuuint64_t dim[5] = {(cuuint64_t)v.size[4], (cuuint64_t)v.size[3], (cuuint64_t)v.size[2], (cuuint64_t)v.size[1],
                       (cuuint64_t)v.size[0]};
  const int64_t st[5] = {1, v.stride[3], v.stride[2], v.stride[1], v.stride[0]};
  *bcast_g = 0;
  *bcast_b = 0;
  cuuint64_t gstride[4];
  int64_t span = (int64_t)dim[0] * 2;
  for (int i = 1; i < 5; ++i) {
    int64_t bytes = st[i] * 2;
    if (dim[i] <= 1 || st[i] == 0) {
      if (dim[i] > 1) {
        if (i == 3) *bcast_g = 1;
        else if (i == 4) *bcast_b = 1;
        else return fail(FL_ERR_UNSUPPORTED, "stride-0 broadcast of the S or H dim is not supported on the bf16 path");
      }
      dim[i] = 1;
      bytes = (span + 15) / 16 * 16;
    }
    if (bytes <= 0 || bytes % 16 != 0 || bytes >= (1ll << 40))
      return fail(FL_ERR_MISALIGNED, "TMA needs 16-byte multiple strides (dim %d: %lld bytes)", i, (long long)bytes);
    gstride[i - 1] = (cuuint64_t)bytes;
    span = std::max<int64_t>(span, bytes * (int64_t)dim[i]);
  }
  if (reinterpret_cast<uintptr_t>(v.data) % 16 != 0) return fail(FL_ERR_MISALIGNED, "TMA needs 16-byte aligned data");
  cuuint32_t box[5] = {(cuuint32_t)ch, (cuuint32_t)box_rows, 1, 1, 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, v.data, dim, gstride, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, ch == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FL_ERR_CUDA, "cuTensorMapEncodeTiled failed (CUresult %d)", (int)r);
  return FL_OK;
}

struct Prepared {
  AttnParams p{};
  View5 q, k, v, o, lse, bias, gate, km;
  int q_rank = 4;
  size_t keybits_bytes = 0;
  size_t ws_bytes = 0;       // bf16: [0,256) scheduler ticket counter, then the packed key mask,
                             // then (short-query path) the split-KV partials
  bool decode = false;       // bf16 short-query split-KV path (decode.cu)
  size_t decode_off = 0;
  bool empty_work = false;
  bool no_keys = false;
  bool bf16 = false;
};

fl_status check_vec(const fl_tensor& t, int dtype, int64_t n, const char* what) {
  if (!t.data) return FL_OK;
  if (t.dtype != dtype || t.rank != 1 || t.size[0] != n || (n > 1 && t.stride[0] != 1))
    return fail(FL_ERR_INVALID_ARGUMENT, "%s: expected contiguous 1-D tensor of %lld elements", what, (long long)n);
  return FL_OK;
}

fl_status prepare(const fl_attn_args* a, Prepared& P, bool device_ptrs) {
  if (!a) return fail(FL_ERR_INVALID_ARGUMENT, "args is NULL");
  const fl_variant& var = a->var;
  if (var.abi_version != FL_ABI_VERSION)
    return fail(FL_ERR_ABI_VERSION, "abi_version %u != %d", var.abi_version, FL_ABI_VERSION);
  if (!given(a->q) || !given(a->k) || !given(a->v) || !given(a->o))
    return fail(FL_ERR_INVALID_ARGUMENT, "q, k, v and o are required");
  const int R = a->q.rank;
  if (R != 4 && R != 5) return fail(FL_ERR_INVALID_ARGUMENT, "q rank must be 4 or 5");
  P.q_rank = R;
  if (!to_view(a->q, R, 0, P.q) || !to_view(a->k, R, 0, P.k) || !to_view(a->v, R, 0, P.v) ||
      !to_view(a->o, R, 0, P.o))
    return fail(FL_ERR_SHAPE_MISMATCH, "q/k/v/o must share one rank (4 or 5) with non-negative sizes");
  const int dt = a->q.dtype;
  if (dt != FL_BF16 && dt != FL_F32) return fail(FL_ERR_UNSUPPORTED, "q dtype must be bf16 or f32");
  if (a->k.dtype != dt || a->v.dtype != dt || a->o.dtype != dt)
    return fail(FL_ERR_INVALID_ARGUMENT, "q, k, v and o must share one dtype");
  P.bf16 = dt == FL_BF16;
  for (const View5* t : {&P.q, &P.k, &P.v, &P.o})
    if (t->size[4] > 1 && t->stride[4] != 1)
      return fail(FL_ERR_UNSUPPORTED, "the last dim of q/k/v/o must be contiguous");
  const int maps = var.diff ? 2 : 1;
  const int64_t B = P.q.size[0], G = P.q.size[1];
  // paged KV: k / v are page pools [n_pages, H, 128, D]; their batch dim indexes pages
  const bool paged = var.kv_page_table.data != nullptr;
  if (paged) {
    const fl_tensor& t = var.kv_page_table;
    if (!P.bf16 || R != 4) return fail(FL_ERR_UNSUPPORTED, "paged KV: bf16, rank-4 q/k/v/o only");
    if (t.dtype != FL_I32 || t.rank != 2 || t.size[0] != B || t.size[1] < 1 || t.stride[1] != 1)
      return fail(FL_ERR_INVALID_ARGUMENT, "kv_page_table: i32 [B, n_pages] with contiguous rows");
    if (P.k.size[3] != 128 || P.v.size[3] != 128)
      return fail(FL_ERR_SHAPE_MISMATCH, "paged KV: k/v pools are [n_pages, H, 128, D] (128-key pages)");
    if (var.kv_len < 0 || var.kv_len > t.size[1] * 128)
      return fail(FL_ERR_INVALID_ARGUMENT, "paged KV: 0 <= kv_len <= 128 * n_pages_per_seq");
  }
  for (const View5* t : {&P.k, &P.v, &P.o})
    if ((!paged || t == &P.o) && (t->size[0] != B || t->size[1] != G))
      return fail(FL_ERR_SHAPE_MISMATCH, "batch dims of q/k/v/o differ");
  if (P.q.size[2] % maps || P.k.size[2] % maps) return fail(FL_ERR_SHAPE_MISMATCH, "diff: q, k carry 2*H heads");
  const int64_t Hq = P.q.size[2] / maps, Hkv = P.k.size[2] / maps;
  if (P.v.size[2] != Hkv || P.o.size[2] != Hq || Hkv == 0 || Hq % Hkv)
    return fail(FL_ERR_SHAPE_MISMATCH, "heads: need v.H == k.H/maps, o.H == q.H/maps, Hq %% Hkv == 0");
  const int64_t Sq = P.q.size[3], Sk = paged ? (int64_t)var.kv_len : P.k.size[3], Dqk = P.q.size[4], Dv = P.v.size[4];
  if (P.o.size[3] != Sq || P.v.size[3] != P.k.size[3] || P.k.size[4] != Dqk || P.o.size[4] != Dv)
    return fail(FL_ERR_SHAPE_MISMATCH, "q/k/v/o sequence or head-dim sizes disagree");
  if (Sq >= (1ll << 30) || Sk >= (1ll << 30) || B * G * Hq >= (1ll << 30))
    return fail(FL_ERR_UNSUPPORTED, "sizes beyond 2^30");
  if (P.bf16) {
    if (Dqk != Dv || (Dqk != 32 && Dqk != 64 && Dqk != 128))
      return fail(FL_ERR_UNSUPPORTED, "bf16 path: D_qk == D_v in {32, 64, 128} (got %lld, %lld)", (long long)Dqk,
                  (long long)Dv);
  } else if (Dqk < 1 || Dqk > 128 || Dv < 1 || Dv > 128) {
    return fail(FL_ERR_UNSUPPORTED, "f32 path: D_qk, D_v in [1, 128]");
  }
  if (var.mod < FL_MOD_NONE || var.mod > FL_MOD_SOFTCAP) return fail(FL_ERR_INVALID_ARGUMENT, "bad mod");
  if (var.mask < FL_MASK_NONE || var.mask > FL_MASK_BLOCKLIST) return fail(FL_ERR_INVALID_ARGUMENT, "bad mask");
  if (var.gate_mode < FL_GATE_NONE || var.gate_mode > FL_GATE_SIGMOID)
    return fail(FL_ERR_INVALID_ARGUMENT, "bad gate_mode");
  if (var.mod == FL_MOD_SOFTCAP && !(var.softcap > 0.f)) return fail(FL_ERR_INVALID_ARGUMENT, "softcap must be > 0");
  if (var.mod == FL_MOD_ALIBI && check_vec(var.alibi_slopes, FL_F32, Hq, "alibi_slopes")) return FL_ERR_INVALID_ARGUMENT;
  if (var.diff && check_vec(var.lambda_h, FL_F32, Hq, "lambda_h")) return FL_ERR_INVALID_ARGUMENT;
  if ((var.lambda_qk.data || var.diff_norm) && !var.diff)
    return fail(FL_ERR_INVALID_ARGUMENT, "lambda_qk / diff_norm need diff (differential attention)");
  if (var.lambda_qk.data && check_vec(var.lambda_qk, FL_F32, 4 * P.q.size[4], "lambda_qk [4, D_qk]"))
    return FL_ERR_INVALID_ARGUMENT;
  if (var.diff_norm && (var.diff_norm != 1 || !(var.diff_norm_eps > 0.f)))
    return fail(FL_ERR_INVALID_ARGUMENT, "diff_norm is 0 or 1, with diff_norm_eps > 0");
  if (var.diff_norm && var.diff_norm_w.data && check_vec(var.diff_norm_w, FL_F32, P.v.size[4], "diff_norm_w [D_v]"))
    return FL_ERR_INVALID_ARGUMENT;
  if (var.causal_align != 0 && var.causal_align != 1) return fail(FL_ERR_INVALID_ARGUMENT, "causal_align is 0 or 1");
  if (var.mask == FL_MASK_SLIDING && var.window < 0) return fail(FL_ERR_INVALID_ARGUMENT, "window must be >= 0");
  if (var.mask == FL_MASK_PREFIX && var.prefix_len < 0) return fail(FL_ERR_INVALID_ARGUMENT, "prefix_len >= 0");
  int n_docs = 0;
  if (var.mask == FL_MASK_DOCUMENT) {
    const fl_tensor& d = var.doc_offsets;
    if (!d.data || d.dtype != FL_I32 || d.rank != 2 || d.size[0] != B || d.size[1] < 2 || d.stride[1] != 1)
      return fail(FL_ERR_INVALID_ARGUMENT, "doc_offsets: i32 [B, n_docs+1] with contiguous rows");
    n_docs = (int)d.size[1] - 1;
  }
  if (var.mask == FL_MASK_BLOCKLIST) {
    if (var.blk_q <= 0 || var.blk_k <= 0 || var.blk_q % 16 || var.blk_k % 32)
      return fail(FL_ERR_INVALID_ARGUMENT, "blocklist: blk_q % 16 == 0, blk_k % 32 == 0");
    if (P.bf16 && (var.blk_q != 128 || var.blk_k != 128))
      return fail(FL_ERR_UNSUPPORTED, "bf16 blocklist path needs blk_q == blk_k == 128");
    if (P.bf16 && var.blk_idx.data && var.blk_idx.rank == 3 && var.blk_idx.size[2] > 256)
      return fail(FL_ERR_UNSUPPORTED, "bf16 blocklist path: max_sel <= 256");
    if (P.bf16 && (var.diff || var.bias.data))
      return fail(FL_ERR_UNSUPPORTED, "bf16 blocklist path: no diff, no additive bias (RSA lists only)");
    const int64_t nqb = (Sq + var.blk_q - 1) / var.blk_q;
    const fl_tensor &bi = var.blk_idx, &bc = var.blk_cnt;
    if (!bi.data || !bc.data || bi.dtype != FL_I32 || bc.dtype != FL_I32 || bi.rank != 3 || bc.rank != 2 ||
        bi.size[0] != B * G * Hq || bi.size[1] != nqb || bc.size[0] != B * G * Hq || bc.size[1] != nqb ||
        bi.stride[2] != 1 || bi.stride[1] != bi.size[2] || bi.stride[0] != nqb * bi.size[2] || bc.stride[1] != 1 ||
        bc.stride[0] != nqb)
      return fail(FL_ERR_INVALID_ARGUMENT, "blk_idx i32 [B*G*Hq, n_qblk, max_sel], blk_cnt i32 [B*G*Hq, n_qblk], contiguous");
  }
  // optional tensors -------------------------------------------------------
  if (a->lse.data) {
    if (a->lse.dtype != FL_F32) return fail(FL_ERR_INVALID_ARGUMENT, "lse must be f32");
    if (!to_view(a->lse, R, -1, P.lse)) return fail(FL_ERR_SHAPE_MISMATCH, "lse rank must be rank(q)-1");
    if (P.lse.size[0] != B || P.lse.size[1] != G || P.lse.size[2] != Hq || P.lse.size[3] != Sq)
      return fail(FL_ERR_SHAPE_MISMATCH, "lse shape must be [B,(G,)Hq,Sq]");
    if (var.diff) return fail(FL_ERR_INVALID_ARGUMENT, "lse must be absent with diff (two softmax maps)");
  }
  if (var.bias.data) {
    if (var.bias.dtype != FL_BF16 && var.bias.dtype != FL_F32) return fail(FL_ERR_INVALID_ARGUMENT, "bias: bf16 or f32");
    if (!to_view(var.bias, R, 0, P.bias)) return fail(FL_ERR_SHAPE_MISMATCH, "bias rank must equal rank(q)");
    const int64_t want[5] = {B, G, Hq, Sq, Sk};
    for (int i = 0; i < 5; ++i)
      if (P.bias.size[i] != want[i] && !(P.bias.size[i] == 1))
        return fail(FL_ERR_SHAPE_MISMATCH, "bias must broadcast to [B,(G,)Hq,Sq,Sk]");
    for (int i = 0; i < 5; ++i)
      if (P.bias.size[i] == 1 && want[i] > 1) {
        P.bias.size[i] = want[i];
        P.bias.stride[i] = 0;
      }
  }
  if (var.key_mask.data) {
    if (var.key_mask.dtype != FL_U8) return fail(FL_ERR_INVALID_ARGUMENT, "key_mask must be u8");
    if (var.key_mask.rank != R - 2) return fail(FL_ERR_SHAPE_MISMATCH, "key_mask rank must be rank(q)-2");
    P.km.present = true;
    P.km.data = var.key_mask.data;
    P.km.dtype = FL_U8;
    if (R == 5) {
      P.km.size[0] = var.key_mask.size[0]; P.km.stride[0] = var.key_mask.stride[0];
      P.km.size[1] = var.key_mask.size[1]; P.km.stride[1] = var.key_mask.stride[1];
      P.km.size[4] = var.key_mask.size[2]; P.km.stride[4] = var.key_mask.stride[2];
    } else {
      P.km.size[0] = var.key_mask.size[0]; P.km.stride[0] = var.key_mask.stride[0];
      P.km.size[4] = var.key_mask.size[1]; P.km.stride[4] = var.key_mask.stride[1];
    }
    if ((P.km.size[0] != B && P.km.size[0] != 1) || (P.km.size[1] != G && P.km.size[1] != 1) || P.km.size[4] != Sk)
      return fail(FL_ERR_SHAPE_MISMATCH, "key_mask must be [B,(G,)Sk]");
    P.keybits_bytes = (size_t)B * G * ((Sk + 127) / 128) * 16;
  }
  if (var.gate_mode != FL_GATE_NONE) {
    if (!var.gate.data) return fail(FL_ERR_INVALID_ARGUMENT, "gate_mode set but gate absent");
    if (!to_view(var.gate, R, 0, P.gate)) return fail(FL_ERR_SHAPE_MISMATCH, "gate rank must equal rank(q)");
    for (int i = 0; i < 5; ++i)
      if (P.gate.size[i] != P.o.size[i]) return fail(FL_ERR_SHAPE_MISMATCH, "gate shape must equal o's");
    if (P.gate.size[4] > 1 && P.gate.stride[4] != 1) return fail(FL_ERR_UNSUPPORTED, "gate last dim must be contiguous");
    if (P.bf16 && var.gate.dtype != FL_BF16) return fail(FL_ERR_UNSUPPORTED, "bf16 path: gate must be bf16");
    if (!P.bf16 && var.gate.dtype != FL_BF16 && var.gate.dtype != FL_F32)
      return fail(FL_ERR_INVALID_ARGUMENT, "gate must be bf16 or f32");
  }
  // alignment (bf16 path: TMA + 16-byte vector epilogue) -----------------------
  if (P.bf16) {
    for (const View5* t : {&P.q, &P.k, &P.v, &P.o})
      if (!aligned16(*t)) return fail(FL_ERR_MISALIGNED, "bf16 path: q/k/v/o need 16-byte aligned base and strides");
    if (P.gate.present && !aligned16(P.gate)) return fail(FL_ERR_MISALIGNED, "bf16 path: gate needs 16-byte alignment");
  }
  // aliasing: o must not overlap any input
  for (const View5* t : {&P.q, &P.k, &P.v, &P.gate, &P.bias})
    if (overlaps(P.o, *t)) return fail(FL_ERR_INVALID_ARGUMENT, "o overlaps an input tensor");
  if (P.lse.present && (overlaps(P.lse, P.o) || overlaps(P.lse, P.q) || overlaps(P.lse, P.k) || overlaps(P.lse, P.v)))
    return fail(FL_ERR_INVALID_ARGUMENT, "lse overlaps another tensor");
  if (device_ptrs) {
    const void* ptrs[] = {a->q.data, a->k.data, a->v.data, a->o.data, a->lse.data, var.bias.data, var.key_mask.data,
                          var.gate.data, var.alibi_slopes.data, var.lambda_h.data, var.doc_offsets.data,
                          var.blk_idx.data, var.blk_cnt.data, var.kv_page_table.data, var.lambda_qk.data,
                          var.diff_norm_w.data};
    for (const void* p : ptrs)
      if (!on_device(p)) return fail(FL_ERR_INVALID_ARGUMENT, "a tensor pointer is not device memory on this device");
  }

  // device params ------------------------------------------------------------
  AttnParams& p = P.p;
  p.B = (int)B; p.G = (int)G; p.Hq = (int)Hq; p.Hkv = (int)Hkv; p.Sq = (int)Sq; p.Sk = (int)Sk;
  p.Dqk = (int)Dqk; p.Dv = (int)Dv; p.maps = maps; p.grp = (int)(Hq / Hkv);
  p.q_off = var.causal_align ? 0 : (int)(Sk - Sq);
  p.q = P.q.data; p.k = P.k.data; p.v = P.v.data; p.o = P.o.data;
  p.qs = strides_of(P.q); p.ks = strides_of(P.k); p.vs = strides_of(P.v); p.os = strides_of(P.o);
  p.lse = static_cast<float*>(P.lse.data); p.lses = strides_of(P.lse);
  p.scale = var.scale != 0.f ? var.scale : 1.f / std::sqrt((float)Dqk);
  p.scale_log2 = p.scale * 1.4426950408889634f;
  p.mod = var.mod; p.softcap = var.softcap;
  p.alibi = static_cast<const float*>(var.alibi_slopes.data);
  p.mask = var.mask; p.window = var.window; p.prefix = var.prefix_len;
  p.doc_offsets = static_cast<const int32_t*>(var.doc_offsets.data); p.n_docs = n_docs;
  p.doc_stride_b = var.mask == FL_MASK_DOCUMENT ? var.doc_offsets.stride[0] : 0;
  p.doc_causal = var.doc_causal;
  p.bias = P.bias.data; p.bias_dtype = P.bias.present ? (P.bias.dtype == FL_F32 ? 1 : 0) : 0;
  p.bs = strides_of(P.bias);
  p.bias_vec = P.bias.present && P.bias.dtype == FL_BF16 && P.bias.stride[4] == 1 &&
               reinterpret_cast<uintptr_t>(P.bias.data) % 16 == 0 && (p.bs.b * 2) % 16 == 0 &&
               (p.bs.g * 2) % 16 == 0 && (p.bs.h * 2) % 16 == 0 && (p.bs.s * 2) % 16 == 0;
  p.keybits = nullptr; p.keybits_words = (int)((Sk + 127) / 128) * 4;
  p.gate_mode = var.gate_mode; p.gate = P.gate.data; p.gs = strides_of(P.gate);
  p.gate_dtype = P.gate.present ? (P.gate.dtype == FL_F32 ? 1 : 0) : 0;
  p.lambda = var.lambda; p.lambda_h = static_cast<const float*>(var.lambda_h.data);
  p.lambda_qk = static_cast<const float*>(var.lambda_qk.data); p.lambda_init = var.lambda_init;
  p.diff_norm = var.diff_norm; p.diff_norm_eps = var.diff_norm_eps;
  p.diff_norm_w = static_cast<const float*>(var.diff_norm_w.data);
  p.blk_idx = static_cast<const int32_t*>(var.blk_idx.data); p.blk_cnt = static_cast<const int32_t*>(var.blk_cnt.data);
  p.blk_q = var.blk_q; p.blk_k = var.blk_k;
  p.max_sel = var.mask == FL_MASK_BLOCKLIST ? (int)var.blk_idx.size[2] : 0;
  p.n_qblk = var.mask == FL_MASK_BLOCKLIST ? (int)((Sq + var.blk_q - 1) / var.blk_q) : 0;
  p.page_table = static_cast<const int32_t*>(var.kv_page_table.data);
  p.page_stride = paged ? var.kv_page_table.stride[0] : 0;
  p.in_dtype = P.bf16 ? 0 : 1;
  // Short query blocks (decode, S_q <= 16): split-KV kernels instead of 128-row tensor-core tiles.
  P.decode = P.bf16 && Sq <= 16 && maps == 1 && !P.bias.present && var.gate_mode == FL_GATE_NONE &&
             Dqk == Dv && (Dqk == 64 || Dqk == 128) && (var.mask != FL_MASK_BLOCKLIST || var.blk_k == 128);
  P.ws_bytes = (P.bf16 ? kSchedBytes : 0) + ((P.keybits_bytes + 255) & ~size_t(255));
  P.decode_off = P.ws_bytes;
  if (P.decode) P.ws_bytes += (decode_workspace_bytes(p, device_sm_count()) + 255) & ~size_t(255);
  P.empty_work = B * G * Hq * Sq == 0 || Dv == 0;
  P.no_keys = Sk == 0;
  return FL_OK;
}

fl_status launch_prepared(Prepared& P, const fl_attn_args* a) {
  cudaStream_t stream = static_cast<cudaStream_t>(a->stream);
  if (P.empty_work) return FL_OK;
  cudaError_t e;
  if (P.no_keys) {
    e = launch_fill_empty(P.p, stream);
    ++g_launches;
    return e == cudaSuccess ? FL_OK : cuda_fail(e, "fill_empty launch");
  }
  TmaMaps maps;
  memset(&maps, 0, sizeof maps);
  if (P.bf16) {
    const int ch = tc_chunk_elems(P.p.Dqk);
    fl_status s;
    if ((s = encode_map(P.q, ch, &maps.q, &maps.q_bcast_g, &maps.q_bcast_b)) != FL_OK) return s;
    if ((s = encode_map(P.k, ch, &maps.k, &maps.k_bcast_g, &maps.k_bcast_b)) != FL_OK) return s;
    if ((s = encode_map(P.v, ch, &maps.v, &maps.v_bcast_g, &maps.v_bcast_b)) != FL_OK) return s;
    // D = 32 kernels stage bf16 bias tiles through TMA when the view allows it (else: direct loads)
    if (P.bias.present && P.p.bias_vec && P.p.Dqk == 32 && !P.decode) {
      const std::string saved = g_err;
      maps.bias_tma = encode_map(P.bias, 64, &maps.bias, &maps.bias_bcast_g, &maps.bias_bcast_b) == FL_OK;
      g_err = saved;
    }
  }
  if (P.ws_bytes && (!a->workspace || a->workspace_bytes < P.ws_bytes))
    return fail(FL_ERR_WORKSPACE, "this call needs %zu bytes of workspace (fl_attn_workspace_size)", P.ws_bytes);
  if (P.bf16) {
    P.p.tile_ctr = static_cast<int32_t*>(a->workspace);
    e = cudaMemsetAsync(P.p.tile_ctr, 0, sizeof(int32_t), stream);
    if (e != cudaSuccess) return cuda_fail(e, "scheduler counter reset");
  }
  if (P.km.present) {
    uint32_t* bits = reinterpret_cast<uint32_t*>(static_cast<char*>(a->workspace) + (P.bf16 ? kSchedBytes : 0));
    e = launch_pack_keymask(static_cast<const unsigned char*>(P.km.data), P.km.size[0] > 1 ? P.km.stride[0] : 0,
                            P.km.size[1] > 1 ? P.km.stride[1] : 0, P.km.stride[4], P.p.B, P.p.G, P.p.Sk,
                            P.p.keybits_words, bits, stream);
    ++g_launches;
    if (e != cudaSuccess) return cuda_fail(e, "pack_keymask launch");
    P.p.keybits = bits;
  }
  if (P.bf16 && P.decode) {
    e = launch_attn_decode(P.p, maps, reinterpret_cast<float*>(static_cast<char*>(a->workspace) + P.decode_off),
                           device_sm_count(), stream);
    ++g_launches;                                       // split + combine
  } else if (P.bf16) {
    e = launch_attn_tc(P.p, maps, stream);
  } else {
    e = launch_attn_simt(P.p, stream);
  }
  ++g_launches;
  return e == cudaSuccess ? FL_OK : cuda_fail(e, "attention launch");
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

// =============================================================================== C ABI
extern "C" {

fl_status fl_attn_fwd(const fl_attn_args* args) {
  Prepared P;
  fl_status s = prepare(args, P, true);
  if (s != FL_OK) return s;
  return launch_prepared(P, args);
}

fl_status fl_attn_workspace_size(const fl_attn_args* args, size_t* bytes) {
  if (!bytes) return fail(FL_ERR_INVALID_ARGUMENT, "bytes is NULL");
  Prepared P;
  fl_status s = prepare(args, P, false);
  if (s != FL_OK) return s;
  *bytes = P.empty_work || P.no_keys ? 0 : P.ws_bytes;
  return FL_OK;
}

// ---- host-buffer (end-to-end) entry --------------------------------------------
namespace {
struct HostPlan {
  struct Item {
    fl_tensor* t;       // tensor in the device copy of the args
    size_t bytes;
    size_t off;
    bool out;
  };
  Item items[20];
  int n = 0;
  size_t total = 0;
  size_t ws_off = 0, ws_bytes = 0;
};

size_t dense_bytes(const fl_tensor& t) {
  size_t n = 1;
  for (int i = 0; i < t.rank; ++i) n *= (size_t)t.size[i];
  return n * elem_bytes(t.dtype);
}

bool is_contiguous(const fl_tensor& t) {
  int64_t expect = 1;
  for (int i = t.rank - 1; i >= 0; --i) {
    if (t.size[i] > 1 && t.stride[i] != expect) return false;
    expect *= t.size[i];
  }
  return true;
}

fl_status plan_host(fl_attn_args& d, HostPlan& hp) {
  fl_tensor* ins[] = {&d.q, &d.k, &d.v, &d.var.bias, &d.var.key_mask, &d.var.gate, &d.var.alibi_slopes,
                      &d.var.lambda_h, &d.var.doc_offsets, &d.var.blk_idx, &d.var.blk_cnt, &d.var.kv_page_table,
                      &d.var.lambda_qk, &d.var.diff_norm_w};
  for (fl_tensor* t : ins) {
    if (!t->data) continue;
    if (!is_contiguous(*t)) return fail(FL_ERR_UNSUPPORTED, "fl_attn_fwd_host: host tensors must be contiguous");
    hp.items[hp.n++] = {t, dense_bytes(*t), hp.total, false};
    hp.total = align256(hp.total + dense_bytes(*t));
  }
  fl_tensor* outs[] = {&d.o, &d.lse};
  for (fl_tensor* t : outs) {
    if (!t->data) continue;
    if (!is_contiguous(*t)) return fail(FL_ERR_UNSUPPORTED, "fl_attn_fwd_host: host tensors must be contiguous");
    hp.items[hp.n++] = {t, dense_bytes(*t), hp.total, true};
    hp.total = align256(hp.total + dense_bytes(*t));
  }
  return FL_OK;
}
}  // namespace

fl_status fl_attn_host_scratch_size(const fl_attn_args* args, size_t* bytes) {
  if (!args || !bytes) return fail(FL_ERR_INVALID_ARGUMENT, "NULL argument");
  fl_attn_args d = *args;
  HostPlan hp;
  fl_status s = plan_host(d, hp);
  if (s != FL_OK) return s;
  Prepared P;
  if ((s = prepare(args, P, false)) != FL_OK) return s;
  *bytes = hp.total + P.ws_bytes;
  return FL_OK;
}

fl_status fl_attn_fwd_host(const fl_attn_args* host_args, void* scratch, size_t scratch_bytes) {
  if (!host_args) return fail(FL_ERR_INVALID_ARGUMENT, "args is NULL");
  fl_attn_args d = *host_args;
  HostPlan hp;
  fl_status s = plan_host(d, hp);
  if (s != FL_OK) return s;
  Prepared P0;
  if ((s = prepare(host_args, P0, false)) != FL_OK) return s;
  const size_t need = hp.total + P0.ws_bytes;
  if (!scratch || scratch_bytes < need) return fail(FL_ERR_WORKSPACE, "fl_attn_fwd_host needs %zu scratch bytes", need);
  if (!on_device(scratch)) return fail(FL_ERR_INVALID_ARGUMENT, "scratch must be device memory");
  cudaStream_t stream = static_cast<cudaStream_t>(host_args->stream);
  char* base = static_cast<char*>(scratch);
  void* host_ptr[16];
  for (int i = 0; i < hp.n; ++i) {
    host_ptr[i] = hp.items[i].t->data;
    hp.items[i].t->data = base + hp.items[i].off;
    // re-stride as dense row-major (same layout as the contiguous host tensor)
  }
  d.workspace = base + hp.total;
  d.workspace_bytes = P0.ws_bytes;
  // Pipelined over batch chunks when only q / k / v (+ small per-call vectors) carry the batch: chunk c's
  // H2D (copy-in stream), kernel (the caller's stream) and D2H (copy-out stream) overlap with the other
  // chunks' transfers; events order them, and the caller's stream waits for the last D2H.
  const int64_t B = host_args->q.rank >= 4 ? host_args->q.size[0] : 1;
  const bool chunkable = B >= 2 && !d.var.bias.data && !d.var.key_mask.data && !d.var.gate.data &&
                         !d.var.blk_idx.data && !d.var.kv_page_table.data && d.k.size[0] == B && d.v.size[0] == B &&
                         d.o.size[0] == B && (!d.lse.data || d.lse.size[0] == B) &&
                         (!d.var.doc_offsets.data || d.var.doc_offsets.size[0] == B);
  if (chunkable) {
    int dev = 0;
    cudaGetDevice(&dev);
    static cudaStream_t s_in[16], s_out[16];
    static std::once_flag once[16];
    if (dev < 0 || dev >= 16) dev = 0;
    std::call_once(once[dev], [&] {
      cudaStreamCreateWithFlags(&s_in[dev], cudaStreamNonBlocking);
      cudaStreamCreateWithFlags(&s_out[dev], cudaStreamNonBlocking);
    });
    constexpr int kMaxChunks = 8;                    // finer chunks shorten the pipeline's fill and drain
    const int nch = (int)std::min<int64_t>(B, kMaxChunks);
    cudaEvent_t ev[2 * kMaxChunks + 2];
    for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventRecord(ev[0], stream);                  // the streams start after the caller's prior work
    cudaStreamWaitEvent(s_in[dev], ev[0], 0);
    cudaStreamWaitEvent(s_out[dev], ev[0], 0);
    // small inputs (no batch dim) once, in full
    for (int i = 0; i < hp.n; ++i) {
      fl_tensor* t = hp.items[i].t;
      if (hp.items[i].out || t == &d.q || t == &d.k || t == &d.v || t == &d.var.doc_offsets) continue;
      cudaMemcpyAsync(t->data, host_ptr[i], hp.items[i].bytes, cudaMemcpyHostToDevice, s_in[dev]);
    }
    fl_status st = FL_OK;
    for (int c = 0; c < nch && st == FL_OK; ++c) {
      const int64_t b0 = B * c / nch, b1 = B * (c + 1) / nch, nb = b1 - b0;
      fl_attn_args dc = d;
      for (int i = 0; i < hp.n; ++i) {
        fl_tensor* t = hp.items[i].t;
        const bool batched = t == &d.q || t == &d.k || t == &d.v || t == &d.var.doc_offsets || t == &d.o || t == &d.lse;
        if (!batched) continue;
        const size_t row = hp.items[i].bytes / (size_t)B;    // bytes per batch entry (contiguous, batch-major)
        char* dptr = static_cast<char*>(t->data) + row * b0;
        // the chunk's view: same tensor, batch range [b0, b1)
        fl_tensor* ct = t == &d.q ? &dc.q : t == &d.k ? &dc.k : t == &d.v ? &dc.v : t == &d.o ? &dc.o
                      : t == &d.lse ? &dc.lse : &dc.var.doc_offsets;
        ct->data = dptr;
        ct->size[0] = nb;
        if (!hp.items[i].out)
          cudaMemcpyAsync(dptr, static_cast<char*>(host_ptr[i]) + row * b0, row * nb, cudaMemcpyHostToDevice, s_in[dev]);
      }
      cudaEventRecord(ev[1 + c], s_in[dev]);
      cudaStreamWaitEvent(stream, ev[1 + c], 0);
      Prepared Pc;
      if ((st = prepare(&dc, Pc, true)) == FL_OK) st = launch_prepared(Pc, &dc);
      cudaEventRecord(ev[1 + nch + c], stream);
      cudaStreamWaitEvent(s_out[dev], ev[1 + nch + c], 0);
      for (int i = 0; i < hp.n; ++i) {
        if (!hp.items[i].out) continue;
        const size_t row = hp.items[i].bytes / (size_t)B;
        cudaMemcpyAsync(static_cast<char*>(host_ptr[i]) + row * b0, static_cast<char*>(hp.items[i].t->data) + row * b0,
                        row * nb, cudaMemcpyDeviceToHost, s_out[dev]);
      }
    }
    cudaEventRecord(ev[2 * nch + 1], s_out[dev]);
    cudaStreamWaitEvent(stream, ev[2 * nch + 1], 0);   // the call's completion is visible on the caller's stream
    for (auto& e : ev) cudaEventDestroy(e);          // deferred by the runtime until the events complete
    if (st != FL_OK) return st;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? FL_OK : cuda_fail(e, "pipelined host call");
  }
  Prepared P;
  if ((s = prepare(&d, P, true)) != FL_OK) return s;
  for (int i = 0; i < hp.n; ++i) {
    if (hp.items[i].out) continue;
    cudaError_t e = cudaMemcpyAsync(hp.items[i].t->data, host_ptr[i], hp.items[i].bytes, cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
  }
  if ((s = launch_prepared(P, &d)) != FL_OK) return s;
  for (int i = 0; i < hp.n; ++i) {
    if (!hp.items[i].out) continue;
    cudaError_t e = cudaMemcpyAsync(host_ptr[i], hp.items[i].t->data, hp.items[i].bytes, cudaMemcpyDeviceToHost, stream);
    if (e != cudaSuccess) return cuda_fail(e, "D2H copy");
  }
  return FL_OK;
}

void fl_shard_range(int64_t units, int32_t world, int32_t rank, int64_t* begin, int64_t* end) {
  if (world <= 0 || rank < 0 || rank >= world || units <= 0) {
    if (begin) *begin = 0;
    if (end) *end = 0;
    return;
  }
  const int64_t base = units / world, rem = units % world;
  const int64_t b = rank * base + std::min<int64_t>(rank, rem);
  if (begin) *begin = b;
  if (end) *end = b + base + (rank < rem ? 1 : 0);
}

fl_status fl_diag_umma_gemm(const void* a, const void* b, float* c, int32_t n, int32_t k, int32_t b_mn_major,
                            int32_t a_from_tmem, void* stream) {
  if (!a || !b || !c) return fail(FL_ERR_INVALID_ARGUMENT, "NULL pointer");
  if ((n != 32 && n != 64 && n != 128) || (k != 32 && k != 64 && k != 128))
    return fail(FL_ERR_UNSUPPORTED, "n, k in {32, 64, 128}");
  View5 va, vb;
  va.present = vb.present = true;
  va.data = const_cast<void*>(a);
  vb.data = const_cast<void*>(b);
  va.dtype = vb.dtype = FL_BF16;
  // A [128, K] row-major
  va.size[3] = 128; va.size[4] = k; va.stride[3] = k; va.stride[4] = 1;
  // B [N, K] (K-major) or [K, N] (MN-major); box rows = 128 covers N or K (OOB rows zero-filled, unused)
  if (b_mn_major) { vb.size[3] = k; vb.size[4] = n; vb.stride[3] = n; }
  else { vb.size[3] = n; vb.size[4] = k; vb.stride[3] = k; }
  vb.stride[4] = 1;
  CUtensorMap ta, tb;
  int g0, b0;
  fl_status s;
  if ((s = encode_map(va, k >= 64 ? 64 : 32, &ta, &g0, &b0)) != FL_OK) return s;
  if ((s = encode_map(vb, b_mn_major ? (n >= 64 ? 64 : 32) : (k >= 64 ? 64 : 32), &tb, &g0, &b0,
                      b_mn_major ? k : n)) != FL_OK)
    return s;
  cudaError_t e = launch_diag_gemm(n, k, ta, tb, a, c, b_mn_major != 0, a_from_tmem != 0, static_cast<cudaStream_t>(stream));
  ++g_launches;
  return e == cudaSuccess ? FL_OK : cuda_fail(e, "diag gemm launch");
}

fl_status fl_debug_schedule(const fl_attn_args* args, int32_t* out, int64_t out_words, int64_t* n_records,
                            int32_t* max_tiles) {
  if (!args || !n_records || !max_tiles) return fail(FL_ERR_INVALID_ARGUMENT, "NULL argument");
  Prepared P;
  fl_status s = prepare(args, P, true);
  if (s != FL_OK) return s;
  if (!P.bf16 || P.decode || P.p.mask == MASK_BLOCKLIST || P.empty_work || P.no_keys)
    return fail(FL_ERR_UNSUPPORTED, "schedule dump covers the bf16 tcgen05 path with interval masks");
  cudaError_t e = launch_sched_dump(P.p, out, out_words, n_records, max_tiles, static_cast<cudaStream_t>(args->stream));
  if (out) ++g_launches;
  if (e == cudaErrorInvalidValue) return fail(FL_ERR_WORKSPACE, "out needs n_records * (8 + max_tiles) words");
  return e == cudaSuccess ? FL_OK : cuda_fail(e, "schedule dump launch");
}

namespace {
struct BwdPrepared {
  Prepared P;
  View5 dout, dq, dk, dv, dgate, dbias;
  size_t ws = 0, off_bits = 0, off_da = 0, off_aun = 0, off_fws = 0, fws = 0;
  fl_attn_args fwd_ungated;         // mul gate: the forward without the gate, recomputing A into the workspace
  int64_t dbias_span = 0;
};

fl_status prepare_bwd(const fl_attn_bwd_args* a, BwdPrepared& B, bool device_ptrs) {
  if (!a) return fail(FL_ERR_INVALID_ARGUMENT, "args is NULL");
  fl_attn_args f;
  memset(&f, 0, sizeof f);
  f.q = a->q; f.k = a->k; f.v = a->v; f.o = a->o; f.lse = a->lse; f.var = a->var;
  f.stream = a->stream;
  fl_status s = prepare(&f, B.P, device_ptrs);
  if (s != FL_OK) return s;
  const fl_variant& var = a->var;
  const AttnParams& p = B.P.p;
  if (!B.P.bf16) return fail(FL_ERR_UNSUPPORTED, "backward: bf16 q/k/v/o");
  if (p.Dqk != 32 && p.Dqk != 64 && p.Dqk != 128) return fail(FL_ERR_UNSUPPORTED, "backward: D in {32, 64, 128}");
  if (var.diff || var.kv_page_table.data || var.mask == FL_MASK_BLOCKLIST)
    return fail(FL_ERR_UNSUPPORTED, "backward: no block list / paged KV");
  if (!a->lse.data && !B.P.empty_work) return fail(FL_ERR_INVALID_ARGUMENT, "backward needs the forward's lse");
  const int R = B.P.q_rank;
  const fl_tensor* ts[4] = {&a->dout, &a->dq, &a->dk, &a->dv};
  View5* vs[4] = {&B.dout, &B.dq, &B.dk, &B.dv};
  const View5* like[4] = {&B.P.o, &B.P.q, &B.P.k, &B.P.v};
  for (int i = 0; i < 4; ++i) {
    if (!given(*ts[i]) || ts[i]->dtype != FL_BF16) return fail(FL_ERR_INVALID_ARGUMENT, "dout / dq / dk / dv: bf16, required");
    if (!to_view(*ts[i], R, 0, *vs[i])) return fail(FL_ERR_SHAPE_MISMATCH, "dout / dq / dk / dv must have q's rank");
    for (int d = 0; d < 5; ++d)
      if (vs[i]->size[d] != like[i]->size[d]) return fail(FL_ERR_SHAPE_MISMATCH, "dout / dq / dk / dv shapes must match o / q / k / v");
    if (vs[i]->stride[4] != 1 || !aligned16(*vs[i])) return fail(FL_ERR_MISALIGNED, "dout / dq / dk / dv: contiguous last dim, 16-byte aligned");
  }
  // dgate (optional; sigmoid gate only): bf16, the gate's shape
  if (a->dgate.data) {
    if (var.gate_mode == FL_GATE_NONE) return fail(FL_ERR_INVALID_ARGUMENT, "dgate needs a gate");
    if (a->dgate.dtype != FL_BF16 || !to_view(a->dgate, R, 0, B.dgate))
      return fail(FL_ERR_SHAPE_MISMATCH, "dgate: bf16 with q's rank");
    for (int d = 0; d < 5; ++d)
      if (B.dgate.size[d] != B.P.o.size[d]) return fail(FL_ERR_SHAPE_MISMATCH, "dgate must have o's shape");
    if (B.dgate.stride[4] != 1 || !aligned16(B.dgate)) return fail(FL_ERR_MISALIGNED, "dgate: contiguous last dim, 16-byte aligned");
  }
  // dbias (optional, with a bias): f32 with the bias's shape; its stride-0 (broadcast) dims accumulate. It must
  // be compact (no gaps between its elements) because the call zeroes its span before the atomics.
  if (a->dbias.data) {
    if (!var.bias.data) return fail(FL_ERR_INVALID_ARGUMENT, "dbias needs a bias");
    if (a->dbias.dtype != FL_F32 || a->dbias.rank != var.bias.rank)
      return fail(FL_ERR_SHAPE_MISMATCH, "dbias: f32 with the bias's rank");
    for (int d = 0; d < a->dbias.rank; ++d)
      if (a->dbias.size[d] != var.bias.size[d]) return fail(FL_ERR_SHAPE_MISMATCH, "dbias must have the bias's shape");
    if (!to_view(a->dbias, R, 0, B.dbias)) return fail(FL_ERR_SHAPE_MISMATCH, "dbias rank");
    int64_t want_span = 1, span = 1;
    for (int d = 0; d < 5; ++d) {
      if (B.dbias.size[d] == 1) B.dbias.stride[d] = 0;
      if (B.dbias.size[d] > 1 && B.dbias.stride[d] != 0) want_span *= B.dbias.size[d];
      if (B.dbias.stride[d] < 0) return fail(FL_ERR_UNSUPPORTED, "dbias: negative strides");
      span += (B.dbias.size[d] - 1) * B.dbias.stride[d];
    }
    if (span != want_span) return fail(FL_ERR_UNSUPPORTED, "dbias must be compact (its span is zeroed by the call)");
    for (int d = 0; d < 5; ++d)                      // the kernel indexes it in the bias's broadcast form
      if (B.dbias.size[d] != B.P.bias.size[d] && B.dbias.size[d] == 1) B.dbias.size[d] = B.P.bias.size[d];
    B.dbias_span = span;
  }
  for (int i = 1; i < 4; ++i)
    for (const View5* in : {&B.P.q, &B.P.k, &B.P.v, &B.P.o, &B.dout, &B.P.gate})
      if (overlaps(*vs[i], *in)) return fail(FL_ERR_INVALID_ARGUMENT, "gradients must not overlap inputs");
  if (B.dgate.present)
    for (const View5* in : {&B.P.q, &B.P.k, &B.P.v, &B.P.o, &B.dout, &B.P.gate, &B.dq, &B.dk, &B.dv})
      if (overlaps(B.dgate, *in)) return fail(FL_ERR_INVALID_ARGUMENT, "dgate must not overlap inputs / gradients");
  if (device_ptrs) {
    for (int i = 0; i < 4; ++i)
      if (!on_device(ts[i]->data)) return fail(FL_ERR_INVALID_ARGUMENT, "dout / dq / dk / dv must be device memory");
    if (!on_device(a->dgate.data)) return fail(FL_ERR_INVALID_ARGUMENT, "dgate must be device memory");
    if (!on_device(a->dbias.data)) return fail(FL_ERR_INVALID_ARGUMENT, "dbias must be device memory");
  }
  // workspace: Dvec f32 [B,G,Hq,Sq] | packed key mask | dO * s(g) bf16 [B,G,Hq,Sq,Dv] (sigmoid gate)
  B.ws = ((size_t)p.B * p.G * p.Hq * p.Sq * sizeof(float) + 255) & ~size_t(255);
  B.off_bits = B.ws;
  B.ws += (B.P.keybits_bytes + 255) & ~size_t(255);
  B.off_da = B.ws;
  if (var.gate_mode != FL_GATE_NONE) B.ws += ((size_t)p.B * p.G * p.Hq * p.Sq * p.Dv * 2 + 255) & ~size_t(255);
  if (var.gate_mode == FL_GATE_MUL) {
    // | A = softmax(s) V without the gate (dgate = dO * A; O / G would divide by the gate) | its forward's workspace
    if (p.Dv % 8) return fail(FL_ERR_UNSUPPORTED, "backward, mul gate: D_v %% 8 == 0");
    B.off_aun = B.ws;
    B.ws += ((size_t)p.B * p.G * p.Hq * p.Sq * p.Dv * 2 + 255) & ~size_t(255);
    fl_attn_args& fu = B.fwd_ungated;
    memset(&fu, 0, sizeof fu);
    fu.q = a->q; fu.k = a->k; fu.v = a->v; fu.var = var; fu.stream = a->stream;
    fu.var.gate_mode = FL_GATE_NONE;
    memset(&fu.var.gate, 0, sizeof fu.var.gate);
    fu.o = a->o;                                     // placeholder data for sizing; contiguous A at run time
    fu.o.stride[fu.o.rank - 1] = 1;
    for (int d = fu.o.rank - 2; d >= 0; --d) fu.o.stride[d] = fu.o.stride[d + 1] * fu.o.size[d + 1];
    fl_status st = fl_attn_workspace_size(&fu, &B.fws);
    if (st != FL_OK) return st;
    B.off_fws = B.ws;
    B.ws += (B.fws + 255) & ~size_t(255);
  }
  return FL_OK;
}
}  // namespace

namespace {
fl_status bwd_single(const fl_attn_bwd_args* args, bool grad_accum = false);

// ---- differential attention backward (Listing 4; reading G8): O = gate'(A_0 - lambda_h A_1) is
// linear in the two maps, so the backward is the single-map backward of each map -- map 0 seeded with dO,
// map 1 with dO_1 = -lambda_h dO -- on the maps' own outputs and LSEs, recomputed by the forward kernel
// (the diff forward keeps neither), with dV (and dgate) summed over the maps:
//   1. fwd(q_i, k_i, v) -> o_i, lse_i            (i = 0, 1; map i = heads [iH, (i+1)H) of q and k)
//   2. dO_1 = -lambda_h dO;  dlambda_h = -sum dO * o_1                 (diff_bwd_seed_kernel)
//   3. bwd(map 0, dO) -> dq[:, :H], dk[:, :Hkv], dv, dgate
//   4. bwd(map 1, dO_1) -> dq[:, H:], dk[:, Hkv:]; dv += (fp32 add in the dK/dV epilogue), dgate += (pre-pass)
fl_tensor head_slice(fl_tensor t, int64_t h0, int64_t nh) {
  const int hd = t.rank - 3;
  if (t.data) t.data = static_cast<char*>(t.data) + h0 * t.stride[hd] * elem_bytes(t.dtype);   // (NULL: empty)
  t.size[hd] = nh;
  return t;
}

fl_tensor dense_like(const fl_tensor& like, void* data, int dtype, int rank) {
  fl_tensor t;
  memset(&t, 0, sizeof t);
  t.data = data; t.dtype = dtype; t.rank = rank;
  int64_t st = 1;
  for (int d = rank - 1; d >= 0; --d) {
    t.size[d] = like.size[d];
    t.stride[d] = st;
    st *= like.size[d];
  }
  return t;
}

size_t up256(size_t x) { return (x + 255) & ~size_t(255); }

struct DiffBwdPlan {
  fl_attn_args fwd[2];
  fl_attn_bwd_args bwd[2];
  AttnParams seed;                  // shape and lambda for the seed kernel
  char* base = nullptr;
  size_t off_do1 = 0, ws = 0;
  bool empty = false;
};

fl_status plan_diff_bwd(const fl_attn_bwd_args* a, DiffBwdPlan& D, bool device_ptrs) {
  const fl_variant& var = a->var;
  if (var.diff_norm) return fail(FL_ERR_UNSUPPORTED, "backward: diff_norm (the G8b RMSNorm epilogue) is not differentiated");
  if (a->dbias.data) return fail(FL_ERR_UNSUPPORTED, "backward: dbias with diff");
  if (var.kv_page_table.data || var.mask == FL_MASK_BLOCKLIST || var.gate_mode == FL_GATE_MUL)
    return fail(FL_ERR_UNSUPPORTED, "backward: no block list / paged KV / mul gate");
  if (a->lse.data) return fail(FL_ERR_INVALID_ARGUMENT, "diff backward: lse must be absent (the maps' LSEs are recomputed)");
  fl_attn_args f;
  memset(&f, 0, sizeof f);
  f.q = a->q; f.k = a->k; f.v = a->v; f.o = a->o; f.var = var; f.stream = a->stream;
  Prepared P;
  fl_status s = prepare(&f, P, device_ptrs);        // validates the diff problem (lambda_h, lambda_qk, ...)
  if (s != FL_OK) return s;
  if (!P.bf16) return fail(FL_ERR_UNSUPPORTED, "backward: bf16 q/k/v/o");
  const AttnParams& p = P.p;
  D.seed = p;
  D.empty = P.empty_work;
  const int64_t Hq = p.Hq, Hkv = p.Hkv;
  const int64_t rows = (int64_t)p.B * p.G * Hq * p.Sq;
  if (p.Dv % 8) return fail(FL_ERR_UNSUPPORTED, "diff backward: D_v %% 8 == 0");
  if (a->dlambda.data) {
    const fl_tensor& t = a->dlambda;
    if (t.dtype != FL_F32 || t.rank != 1 || t.size[0] != Hq || (Hq > 1 && t.stride[0] != 1))
      return fail(FL_ERR_SHAPE_MISMATCH, "dlambda: f32 [Hq], contiguous");
    if (device_ptrs && !on_device(t.data)) return fail(FL_ERR_INVALID_ARGUMENT, "dlambda must be device memory");
  }
  // workspace: o_0 | o_1 | lse_0 | lse_1 | dO_1 | forward workspace | backward workspace
  D.base = device_ptrs ? static_cast<char*>(a->workspace) : reinterpret_cast<char*>(uintptr_t(1) << 12);
  if (!D.base) D.base = reinterpret_cast<char*>(uintptr_t(1) << 12);   // sizes only (checked before running)
  const size_t so = up256((size_t)rows * p.Dv * 2), sl = up256((size_t)rows * 4);
  size_t off = 0;
  const size_t off_o[2] = {0, so}, off_l[2] = {2 * so, 2 * so + sl};
  off = 2 * so + 2 * sl;
  D.off_do1 = off; off += so;
  fl_tensor lse_like = a->o;                          // [B,(G,)Hq,Sq]: o's sizes without the head dim
  lse_like.rank = a->o.rank - 1;
  for (int m = 0; m < 2; ++m) {
    fl_attn_args& fm = D.fwd[m];
    fm = f;
    fm.var.diff = 0;
    memset(&fm.var.lambda_h, 0, sizeof fm.var.lambda_h);
    memset(&fm.var.lambda_qk, 0, sizeof fm.var.lambda_qk);
    fm.q = head_slice(a->q, m * Hq, Hq);
    fm.k = head_slice(a->k, m * Hkv, Hkv);
    fm.o = dense_like(a->o, D.base + off_o[m], FL_BF16, a->o.rank);
    fm.lse = dense_like(lse_like, D.base + off_l[m], FL_F32, lse_like.rank);
  }
  size_t fws = 0;
  if ((s = fl_attn_workspace_size(&D.fwd[0], &fws)) != FL_OK) return s;
  const size_t off_fws = off;
  off += up256(fws);
  size_t bws = 0;
  for (int m = 0; m < 2; ++m) {
    fl_attn_bwd_args& bm = D.bwd[m];
    memset(&bm, 0, sizeof bm);
    bm.q = D.fwd[m].q; bm.k = D.fwd[m].k; bm.v = a->v; bm.o = D.fwd[m].o; bm.lse = D.fwd[m].lse;
    bm.var = D.fwd[m].var;
    bm.stream = a->stream;
    bm.dq = head_slice(a->dq, m * Hq, Hq);
    bm.dk = head_slice(a->dk, m * Hkv, Hkv);
    bm.dout = m == 0 ? a->dout : dense_like(a->dout, D.base + D.off_do1, FL_BF16, a->dout.rank);
    bm.dv = a->dv;
    bm.dgate = a->dgate;
    BwdPrepared B;
    if ((s = prepare_bwd(&bm, B, false)) != FL_OK) return s;
    bws = std::max(bws, B.ws);
  }
  const size_t off_bws = off;
  off += up256(bws);
  for (int m = 0; m < 2; ++m) {
    D.fwd[m].workspace = D.base + off_fws; D.fwd[m].workspace_bytes = fws;
    D.bwd[m].workspace = D.base + off_bws; D.bwd[m].workspace_bytes = bws;
  }
  D.ws = off;
  return FL_OK;
}

fl_status bwd_diff(const fl_attn_bwd_args* a) {
  DiffBwdPlan D;
  fl_status s = plan_diff_bwd(a, D, true);
  if (s != FL_OK) return s;
  if (!a->workspace || a->workspace_bytes < D.ws)
    return fail(FL_ERR_WORKSPACE, "the diff backward needs %zu bytes of workspace", D.ws);
  cudaStream_t stream = static_cast<cudaStream_t>(a->stream);
  if (a->dlambda.data) {
    cudaError_t e = cudaMemsetAsync(a->dlambda.data, 0, (size_t)D.seed.Hq * sizeof(float), stream);
    if (e != cudaSuccess) return cuda_fail(e, "dlambda reset");
  }
  if (D.empty) {                                     // no queries: the per-map calls zero dK, dV
    for (int m = 0; m < 2; ++m)
      if ((s = bwd_single(&D.bwd[m], m == 1)) != FL_OK) return s;
    return FL_OK;
  }
  for (int m = 0; m < 2; ++m) {                      // 1. the maps' outputs and LSEs
    Prepared P;
    if ((s = prepare(&D.fwd[m], P, true)) != FL_OK) return s;
    if ((s = launch_prepared(P, &D.fwd[m])) != FL_OK) return s;
  }
  View5 dov;                                          // 2. map-1 seed and dlambda
  to_view(a->dout, a->q.rank, 0, dov);
  cudaError_t e = launch_diff_bwd_seed(D.seed, a->dout.data, strides_of(dov), D.fwd[1].o.data,
                                       D.base + D.off_do1, static_cast<float*>(a->dlambda.data), stream);
  ++g_launches;
  if (e != cudaSuccess) return cuda_fail(e, "diff seed launch");
  for (int m = 0; m < 2; ++m)                         // 3, 4. the single-map backward of each map; the maps
    if ((s = bwd_single(&D.bwd[m], m == 1)) != FL_OK) return s;   // share V (and the gate): map 1 accumulates
  return FL_OK;
}
}  // namespace

fl_status fl_attn_bwd_workspace_size(const fl_attn_bwd_args* args, size_t* bytes) {
  if (!bytes) return fail(FL_ERR_INVALID_ARGUMENT, "bytes is NULL");
  if (args && args->var.diff) {
    DiffBwdPlan D;
    fl_status s = plan_diff_bwd(args, D, false);
    if (s != FL_OK) return s;
    *bytes = D.ws;
    return FL_OK;
  }
  BwdPrepared B;
  fl_status s = prepare_bwd(args, B, false);
  if (s != FL_OK) return s;
  *bytes = B.ws;
  return FL_OK;
}

fl_status fl_attn_bwd(const fl_attn_bwd_args* args) {
  if (args && args->var.diff) return bwd_diff(args);
  if (args && args->dlambda.data) return fail(FL_ERR_INVALID_ARGUMENT, "dlambda needs diff");
  return bwd_single(args);
}

namespace {
fl_status bwd_single(const fl_attn_bwd_args* args, bool grad_accum) {
  BwdPrepared B;
  fl_status s = prepare_bwd(args, B, true);
  if (s != FL_OK) return s;
  B.P.p.grad_accum = grad_accum ? 1 : 0;
  cudaStream_t stream = static_cast<cudaStream_t>(args->stream);
  if (B.P.empty_work || B.P.no_keys) {
    // no queries: dK = dV = 0; no keys: O = 0 (G7), so dQ = 0 and dgate = 0 (dK, dV, dbias are empty)
    const AttnParams& p = B.P.p;
    cudaError_t e = cudaSuccess;
    auto zero = [&](const View5& v, int H, int S, int D, bool shared) {   // shared: summed over diff maps
      if (e == cudaSuccess && v.present && !(shared && grad_accum)) {
        e = launch_zero_rows(v.data, strides_of(v), p.B, p.G, H, S, D, stream);
        ++g_launches;
      }
    };
    if (B.P.empty_work) {
      zero(B.dk, p.Hkv, p.Sk, p.Dqk, false);
      zero(B.dv, p.Hkv, p.Sk, p.Dv, true);
    } else {
      zero(B.dq, p.Hq, p.Sq, p.Dqk, false);
      zero(B.dgate, p.Hq, p.Sq, p.Dv, true);
    }
    return e == cudaSuccess ? FL_OK : cuda_fail(e, "gradient zero fill");
  }
  if (!args->workspace || args->workspace_bytes < B.ws)
    return fail(FL_ERR_WORKSPACE, "the backward needs %zu bytes of workspace", B.ws);
  char* ws = static_cast<char*>(args->workspace);
  AttnParams& p = B.P.p;
  TmaMaps maps;
  memset(&maps, 0, sizeof maps);
  const int ch = tc_chunk_elems(p.Dqk);
  if ((s = encode_map(B.P.q, ch, &maps.q, &maps.q_bcast_g, &maps.q_bcast_b)) != FL_OK) return s;
  if ((s = encode_map(B.P.k, ch, &maps.k, &maps.k_bcast_g, &maps.k_bcast_b)) != FL_OK) return s;
  if ((s = encode_map(B.P.v, ch, &maps.v, &maps.v_bcast_g, &maps.v_bcast_b)) != FL_OK) return s;
  cudaError_t e;
  if (B.P.km.present) {                              // MSA / key mask -> one bit per key (as the forward)
    uint32_t* bits = reinterpret_cast<uint32_t*>(ws + B.off_bits);
    e = launch_pack_keymask(static_cast<const unsigned char*>(B.P.km.data), B.P.km.size[0] > 1 ? B.P.km.stride[0] : 0,
                            B.P.km.size[1] > 1 ? B.P.km.stride[1] : 0, B.P.km.stride[4], p.B, p.G, p.Sk,
                            p.keybits_words, bits, stream);
    ++g_launches;
    if (e != cudaSuccess) return cuda_fail(e, "pack_keymask launch");
    p.keybits = bits;
  }
  // mul gate: A (the ungated output) for dgate = dO * A, recomputed by the forward kernel
  void* aun = nullptr;
  if (p.gate_mode == GATE_MUL) {
    fl_attn_args fu = B.fwd_ungated;
    aun = ws + B.off_aun;
    fu.o.data = aun;
    fu.workspace = ws + B.off_fws;
    fu.workspace_bytes = B.fws;
    Prepared PU;
    if ((s = prepare(&fu, PU, true)) != FL_OK) return s;
    if ((s = launch_prepared(PU, &fu)) != FL_OK) return s;
  }
  // dO as the tcgen05 kernels read it: the caller's, or dO * gate' from the gate pre-pass (contiguous)
  View5 vda = B.dout;
  void* da = nullptr;
  if (p.gate_mode != GATE_NONE) {
    da = ws + B.off_da;
    vda.data = da;
    vda.stride[4] = 1;
    vda.stride[3] = p.Dv;
    vda.stride[2] = (int64_t)p.Sq * p.Dv;
    vda.stride[1] = (int64_t)p.Hq * p.Sq * p.Dv;
    vda.stride[0] = (int64_t)p.G * p.Hq * p.Sq * p.Dv;
  }
  CUtensorMap tdo, tq64, tdo64;
  int bg, bb;
  if ((s = encode_map(vda, ch, &tdo, &bg, &bb)) != FL_OK) return s;
  if ((s = encode_map(vda, ch, &tdo64, &bg, &bb, 64)) != FL_OK) return s;
  if ((s = encode_map(B.P.q, ch, &tq64, &bg, &bb, 64)) != FL_OK) return s;
  float* dvec = reinterpret_cast<float*>(ws);
  if (B.dbias.present) {
    e = cudaMemsetAsync(B.dbias.data, 0, (size_t)B.dbias_span * sizeof(float), stream);
    if (e != cudaSuccess) return cuda_fail(e, "dbias reset");
  }
  e = launch_bwd_prepass(p, B.dout.data, strides_of(B.dout), dvec, da, B.dgate.data, strides_of(B.dgate), aun, stream);
  ++g_launches;
  if (e != cudaSuccess) return cuda_fail(e, "backward pre-pass launch");
  e = launch_attn_bwd(p, maps, tdo, tq64, tdo64, static_cast<const float*>(B.P.lse.data), strides_of(B.P.lse), B.dout.data,
                      strides_of(B.dout), dvec, B.dq.data, strides_of(B.dq), B.dk.data, strides_of(B.dk), B.dv.data,
                      strides_of(B.dv), static_cast<float*>(B.dbias.data), strides_of(B.dbias), stream);
  g_launches += 2;
  return e == cudaSuccess ? FL_OK : cuda_fail(e, "backward launch");
}
}  // namespace

fl_status fl_linear(const fl_linear_args* a) {
  if (!a) return fail(FL_ERR_INVALID_ARGUMENT, "args is NULL");
  const fl_tensor &x = a->x, &w = a->w, &y = a->y;
  if (!x.data || !w.data || !y.data) return fail(FL_ERR_INVALID_ARGUMENT, "linear: x, w, y are required");
  if (x.dtype != FL_BF16 || w.dtype != FL_BF16 || y.dtype != FL_BF16)
    return fail(FL_ERR_INVALID_ARGUMENT, "linear: x, w, y must be bf16");
  if (x.rank != 2 || w.rank != 2 || y.rank != 2) return fail(FL_ERR_SHAPE_MISMATCH, "linear: x, w, y must be rank 2");
  const int64_t M = x.size[0], K = x.size[1], N = w.size[0];
  if (w.size[1] != K || y.size[0] != M || y.size[1] != N)
    return fail(FL_ERR_SHAPE_MISMATCH, "linear: x [M,K], w [N,K], y [M,N]");
  if (K != 64 && K != 128 && K != 192 && K != 256) return fail(FL_ERR_UNSUPPORTED, "linear: K in {64, 128, 192, 256}");
  if (N < 1 || M < 0 || M >= (1ll << 31) || N >= (1ll << 31)) return fail(FL_ERR_SHAPE_MISMATCH, "linear: bad M / N");
  if (x.stride[1] != 1 || w.stride[1] != 1) return fail(FL_ERR_UNSUPPORTED, "linear: x and w need a contiguous last dim");
  const fl_tensor* f32s[3] = {&a->bias, &a->ln_gamma, &a->ln_beta};
  const int64_t want[3] = {N, K, K};
  for (int i = 0; i < 3; ++i)
    if (f32s[i]->data && (f32s[i]->dtype != FL_F32 || f32s[i]->rank != 1 || f32s[i]->size[0] != want[i] ||
                          f32s[i]->stride[0] != 1))
      return fail(FL_ERR_SHAPE_MISMATCH, "linear: bias f32 [N], ln_gamma / ln_beta f32 [K], contiguous");
  if (a->ln_beta.data && !a->ln_gamma.data) return fail(FL_ERR_INVALID_ARGUMENT, "linear: ln_beta needs ln_gamma");
  for (const void* v : {a->ln_gamma.data, a->ln_beta.data})
    if (v && reinterpret_cast<uintptr_t>(v) % 16 != 0)
      return fail(FL_ERR_MISALIGNED, "linear: ln_gamma / ln_beta need 16-byte alignment");
  const void* ptrs[] = {x.data, w.data, y.data, a->bias.data, a->ln_gamma.data, a->ln_beta.data};
  for (const void* p : ptrs)
    if (!on_device(p)) return fail(FL_ERR_INVALID_ARGUMENT, "linear: pointers must be device memory");
  View5 vx, vw, vy;
  vx.present = vw.present = vy.present = true;
  vx.data = x.data; vx.dtype = FL_BF16; vx.size[3] = M; vx.size[4] = K; vx.stride[3] = x.stride[0]; vx.stride[4] = 1;
  vw.data = w.data; vw.dtype = FL_BF16; vw.size[3] = N; vw.size[4] = K; vw.stride[3] = w.stride[0]; vw.stride[4] = 1;
  vy.data = y.data; vy.dtype = FL_BF16; vy.size[3] = M; vy.size[4] = N; vy.stride[3] = y.stride[0];
  vy.stride[4] = y.stride[1];
  if (overlaps(vy, vx) || overlaps(vy, vw)) return fail(FL_ERR_INVALID_ARGUMENT, "linear: y overlaps x or w");
  if (M == 0) return FL_OK;
  CUtensorMap tx, tw;
  int bg, bb;
  fl_status s;
  if ((s = encode_map(vx, 64, &tx, &bg, &bb)) != FL_OK) return s;
  if ((s = encode_map(vw, 64, &tw, &bg, &bb, linear_nt_max())) != FL_OK) return s;   // W box: one tile of rows
  LinParams p;
  p.M = (int)M; p.N = (int)N; p.K = (int)K;
  p.NT = N >= linear_nt_max() ? linear_nt_max() : (int)((N + 15) / 16 * 16);
  p.bias = static_cast<const float*>(a->bias.data);
  p.ln_g = static_cast<const float*>(a->ln_gamma.data);
  p.ln_b = static_cast<const float*>(a->ln_beta.data);
  p.eps = a->ln_eps;
  p.y = y.data;
  p.ys_m = y.stride[0]; p.ys_n = y.stride[1];
  CUtensorMap ty;                                  // (unused: the epilogue stores rows directly; a TMA-store
  memset(&ty, 0, sizeof ty);                       //  epilogue measured slower, profiles/r02_ab.md)
  const int y_tma = 0;
  const cudaError_t e = launch_linear(p, tx, tw, ty, y_tma, static_cast<cudaStream_t>(a->stream));
  ++g_launches;
  return e == cudaSuccess ? FL_OK : cuda_fail(e, "linear launch");
}

namespace {
struct IpaPrepared {
  fl::IpaParams p;
  int64_t N = 0, H = 0, c = 0, Pq = 0, Pv = 0, cz = 0;
  size_t off_qa = 0, off_ka = 0, off_va = 0, off_gv = 0, off_bias = 0, off_o = 0, off_lse = 0, off_a = 0,
         off_attn = 0, total = 0;
};

bool dense(const fl_tensor& t, int rank, const int64_t* sizes, int dtype) {
  if (!t.data || t.rank != rank || t.dtype != dtype) return false;
  int64_t st = 1;
  for (int d = rank - 1; d >= 0; --d) {
    if (t.size[d] != sizes[d]) return false;
    if (t.size[d] > 1 && t.stride[d] != st) return false;
    st *= t.size[d];
  }
  return true;
}

fl_status prepare_ipa(const fl_ipa_args* a, IpaPrepared& P) {
  if (!a) return fail(FL_ERR_INVALID_ARGUMENT, "args is NULL");
  if (!a->q.data || a->q.rank != 3) return fail(FL_ERR_SHAPE_MISMATCH, "ipa: q [N, H, c]");
  P.N = a->q.size[0]; P.H = a->q.size[1]; P.c = a->q.size[2];
  if (!a->qp.data || a->qp.rank != 4 || !a->vp.data || a->vp.rank != 4 || !a->z.data || a->z.rank != 3)
    return fail(FL_ERR_SHAPE_MISMATCH, "ipa: qp / kp [N, H, Pq, 3], vp [N, H, Pv, 3], z [N, N, cz]");
  P.Pq = a->qp.size[2]; P.Pv = a->vp.size[2]; P.cz = a->z.size[2];
  const int64_t N = P.N, H = P.H, c = P.c;
  const int64_t s_nhc[3] = {N, H, c}, s_qp[4] = {N, H, P.Pq, 3}, s_vp[4] = {N, H, P.Pv, 3}, s_R[3] = {N, 3, 3},
                s_t[2] = {N, 3}, s_b[3] = {H, N, N}, s_z[3] = {N, N, P.cz}, s_g[1] = {H}, s_opair[3] = {N, H, P.cz};
  if (!dense(a->q, 3, s_nhc, FL_BF16) || !dense(a->k, 3, s_nhc, FL_BF16) || !dense(a->v, 3, s_nhc, FL_BF16) ||
      !dense(a->qp, 4, s_qp, FL_BF16) || !dense(a->kp, 4, s_qp, FL_BF16) || !dense(a->vp, 4, s_vp, FL_BF16) ||
      !dense(a->R, 3, s_R, FL_F32) || !dense(a->t, 2, s_t, FL_F32) || !dense(a->bias, 3, s_b, FL_BF16) ||
      !dense(a->z, 3, s_z, FL_BF16) || !dense(a->gamma, 1, s_g, FL_F32) || !dense(a->o, 3, s_nhc, FL_BF16) ||
      !dense(a->op, 4, s_vp, FL_F32) || !dense(a->opair, 3, s_opair, FL_BF16))
    return fail(FL_ERR_SHAPE_MISMATCH, "ipa: tensors must be contiguous with the documented shapes and dtypes");
  if (N < 1 || H < 1 || c < 1 || c + 9 * P.Pq + 2 > 64 || P.cz < 8 || P.cz % 8 != 0 || P.Pv < 0 || P.Pv % 4 != 0 ||
      3 * P.Pv > 24)
    return fail(FL_ERR_UNSUPPORTED, "ipa: c + 9 Pq + 2 <= 64, Pv in {0, 4, 8}, cz %% 8 == 0");
  {
    fl::IpaParams ps;
    ps.N = (int)N; ps.H = (int)H;
    if (N > 65535 || ipa_out_smem(ps) > 227 * 1024)
      return fail(FL_ERR_UNSUPPORTED, "ipa: N <= 8600 (a row's probabilities of 6 heads fit shared memory)");
  }
  for (const fl_tensor* t : {&a->q, &a->k, &a->v, &a->qp, &a->kp, &a->vp, &a->R, &a->t, &a->bias, &a->z, &a->gamma,
                             &a->o, &a->op, &a->opair})
    if (!on_device(t->data)) return fail(FL_ERR_INVALID_ARGUMENT, "ipa: pointers must be device memory");
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t off = 0;
  P.off_qa = off; off += up(N * H * 64 * 2);
  P.off_ka = off; off += up(N * H * 64 * 2);
  P.off_va = off; off += up(N * H * 64 * 2);
  P.off_gv = off; off += up(N * H * (P.Pv > 0 ? P.Pv : 1) * 3 * 4);
  P.off_bias = off; off += up(H * N * N * 4);
  P.off_o = off; off += up(N * H * 64 * 2);
  P.off_lse = off; off += up(H * N * 4);
  P.off_a = off; off += up(H * N * N * 4);           // a_ij^h (fp32) for the pair and point outputs
  P.off_attn = off;
  off += 1024 * 1024;                                // the attention call's workspace (ticket counter)
  P.total = off;
  fl::IpaParams& p = P.p;
  p.N = (int)N; p.H = (int)H; p.c = (int)c; p.Pq = (int)P.Pq; p.Pv = (int)P.Pv; p.cz = (int)P.cz;
  p.q = static_cast<const __nv_bfloat16*>(a->q.data); p.k = static_cast<const __nv_bfloat16*>(a->k.data);
  p.qp = static_cast<const __nv_bfloat16*>(a->qp.data); p.kp = static_cast<const __nv_bfloat16*>(a->kp.data);
  p.vp = static_cast<const __nv_bfloat16*>(a->vp.data); p.bias = static_cast<const __nv_bfloat16*>(a->bias.data);
  p.z = static_cast<const __nv_bfloat16*>(a->z.data);
  p.R = static_cast<const float*>(a->R.data); p.t = static_cast<const float*>(a->t.data);
  p.gamma = static_cast<const float*>(a->gamma.data);
  return FL_OK;
}

fl_tensor mk_tensor(void* data, int dtype, std::initializer_list<int64_t> sizes, std::initializer_list<int64_t> strides) {
  fl_tensor t;
  memset(&t, 0, sizeof t);
  t.data = data; t.dtype = dtype; t.rank = (int)sizes.size();
  int i = 0;
  for (int64_t x : sizes) t.size[i++] = x;
  i = 0;
  for (int64_t x : strides) t.stride[i++] = x;
  return t;
}
}  // namespace

fl_status fl_ipa_workspace_size(const fl_ipa_args* args, size_t* bytes) {
  if (!bytes) return fail(FL_ERR_INVALID_ARGUMENT, "bytes is NULL");
  IpaPrepared P;
  fl_status s = prepare_ipa(args, P);
  if (s != FL_OK) return s;
  *bytes = P.total;
  return FL_OK;
}

fl_status fl_ipa_fwd(const fl_ipa_args* args) {
  IpaPrepared P;
  fl_status s = prepare_ipa(args, P);
  if (s != FL_OK) return s;
  if (!args->workspace || args->workspace_bytes < P.total)
    return fail(FL_ERR_WORKSPACE, "ipa needs %zu bytes of workspace (fl_ipa_workspace_size)", P.total);
  char* ws = static_cast<char*>(args->workspace);
  cudaStream_t stream = static_cast<cudaStream_t>(args->stream);
  fl::IpaParams& p = P.p;
  p.qa = reinterpret_cast<__nv_bfloat16*>(ws + P.off_qa);
  p.ka = reinterpret_cast<__nv_bfloat16*>(ws + P.off_ka);
  p.gv = reinterpret_cast<float*>(ws + P.off_gv);
  p.bias_s = reinterpret_cast<__nv_bfloat16*>(ws + P.off_bias);
  const int64_t N = P.N, H = P.H, c = P.c;
  // V' = [v | 0] (64 columns: the attention kernel's D_v = D_qk); its scalar output o = the first c columns
  __nv_bfloat16* va = reinterpret_cast<__nv_bfloat16*>(ws + P.off_va);
  cudaError_t e = cudaMemsetAsync(va, 0, N * H * 64 * 2, stream);
  if (e == cudaSuccess)
    e = cudaMemcpy2DAsync(va, 64 * 2, args->v.data, c * 2, c * 2, N * H, cudaMemcpyDeviceToDevice, stream);
  if (e != cudaSuccess) return cuda_fail(e, "ipa V' staging");
  if ((e = launch_ipa_prep(p, stream)) != cudaSuccess) return cuda_fail(e, "ipa prep launch");
  g_launches += 2;
  // the fused attention forward over the augmented operands: [B=1, H, S=N, 64] views of [N, H, 64]
  fl_attn_args at;
  memset(&at, 0, sizeof at);
  at.var.abi_version = FL_ABI_VERSION;
  at.var.scale = 1.0f;
  at.q = mk_tensor(p.qa, FL_BF16, {1, H, N, 64}, {N * H * 64, 64, H * 64, 1});
  at.k = mk_tensor(p.ka, FL_BF16, {1, H, N, 64}, {N * H * 64, 64, H * 64, 1});
  at.v = mk_tensor(va, FL_BF16, {1, H, N, 64}, {N * H * 64, 64, H * 64, 1});
  void* o64 = ws + P.off_o;
  at.o = mk_tensor(o64, FL_BF16, {1, H, N, 64}, {N * H * 64, 64, H * 64, 1});
  float* lse = reinterpret_cast<float*>(ws + P.off_lse);
  at.lse = mk_tensor(lse, FL_F32, {1, H, N}, {H * N, N, 1});
  at.var.bias = mk_tensor(p.bias_s, FL_BF16, {1, H, N, N}, {H * N * N, N * N, N, 1});
  at.stream = stream;
  at.workspace = ws + P.off_attn;
  at.workspace_bytes = P.total - P.off_attn;
  if ((s = fl_attn_fwd(&at)) != FL_OK) return s;
  // o = the first c columns of O'
  e = cudaMemcpy2DAsync(args->o.data, c * 2, o64, 64 * 2, c * 2, N * H, cudaMemcpyDeviceToDevice, stream);
  if (e != cudaSuccess) return cuda_fail(e, "ipa o copy");
  if ((e = launch_ipa_finish(p, lse, reinterpret_cast<float*>(ws + P.off_a), args->opair.data,
                             static_cast<float*>(args->op.data), stream)) != cudaSuccess)
    return cuda_fail(e, "ipa finish launch");
  g_launches += 2;
  return FL_OK;
}

fl_status fl_diag_pipe_rate(int32_t op, int32_t iters, float* sink, int64_t* ops, void* stream) {
  if (op < 0 || op > 3 || iters <= 0) return fail(FL_ERR_INVALID_ARGUMENT, "op in 0..3, iters > 0");
  if (!sink) return fail(FL_ERR_INVALID_ARGUMENT, "NULL sink");
  const int n = device_sm_count();
  // elementary ops per chain step: ex2.f32 / tanh 1, ex2.bf16x2 2 (packed), FFMA2 1 (4 packed pairs / 8 chains)
  const int64_t per = op == 1 ? 2 : 1;
  if (ops) *ops = (int64_t)n * 512 * 8 * (int64_t)iters * per;
  cudaError_t e = launch_pipe_rate(op, iters, n, sink, static_cast<cudaStream_t>(stream));
  ++g_launches;
  return e == cudaSuccess ? FL_OK : cuda_fail(e, "pipe rate launch");
}

static fl_status rsa_summaries(const fl_tensor* k, fl_tensor* kmin, fl_tensor* kmax, int32_t blk_k, int64_t k_begin,
                               void* stream) {
  if (!k || !kmin || !kmax || !k->data || !kmin->data || !kmax->data)
    return fail(FL_ERR_INVALID_ARGUMENT, "rsa_build_summaries: k, kmin, kmax are required");
  if (blk_k <= 0) return fail(FL_ERR_INVALID_ARGUMENT, "rsa_build_summaries: blk_k must be > 0");
  if (k_begin < 0) return fail(FL_ERR_INVALID_ARGUMENT, "rsa_update_summaries: k_begin must be >= 0");
  if (k->dtype != FL_BF16 || kmin->dtype != FL_BF16 || kmax->dtype != FL_BF16)
    return fail(FL_ERR_UNSUPPORTED, "rsa_build_summaries: bf16 only");
  if (k->rank != 4 && k->rank != 5) return fail(FL_ERR_INVALID_ARGUMENT, "rsa_build_summaries: k rank 4 or 5");
  View5 kv;
  if (!to_view(*k, k->rank, 0, kv)) return fail(FL_ERR_SHAPE_MISMATCH, "rsa_build_summaries: bad k view");
  const int64_t B = kv.size[0], G = kv.size[1], H = kv.size[2], Sk = kv.size[3], D = kv.size[4];
  if (D % 8 || D > 1024 || D < 8) return fail(FL_ERR_UNSUPPORTED, "rsa_build_summaries: D %% 8 == 0, 8 <= D <= 1024");
  if (D > 1 && kv.stride[4] != 1) return fail(FL_ERR_UNSUPPORTED, "rsa_build_summaries: k last dim must be contiguous");
  if (!aligned16(kv)) return fail(FL_ERR_MISALIGNED, "rsa_build_summaries: k needs 16-byte aligned rows");
  const int64_t nkb = (Sk + blk_k - 1) / blk_k;
  for (const fl_tensor* t : {static_cast<const fl_tensor*>(kmin), static_cast<const fl_tensor*>(kmax)})
    if (t->rank != 3 || t->size[0] != B * G * H || t->size[1] != nkb || t->size[2] != D || t->stride[2] != 1 ||
        t->stride[1] != D || t->stride[0] != nkb * D || reinterpret_cast<uintptr_t>(t->data) % 16)
      return fail(FL_ERR_SHAPE_MISMATCH, "rsa_build_summaries: kmin/kmax must be contiguous bf16 [B*G*Hkv, n_kblk, D]");
  for (const void* ptr : {k->data, kmin->data, kmax->data})
    if (!on_device(ptr)) return fail(FL_ERR_INVALID_ARGUMENT, "rsa_build_summaries: pointers must be device memory");
  if (B * G * H == 0 || nkb == 0) return FL_OK;
  if (B * G * H > 65535) return fail(FL_ERR_UNSUPPORTED, "rsa_build_summaries: B*G*H > 65535");
  cudaError_t e = launch_rsa_summaries(kv.data, kv.size[0] > 1 ? kv.stride[0] : 0, kv.size[1] > 1 ? kv.stride[1] : 0,
                                       kv.size[2] > 1 ? kv.stride[2] : 0, kv.stride[3], (int)B, (int)G, (int)H, (int)Sk,
                                       (int)D, blk_k, (int)std::min<int64_t>(k_begin / blk_k, nkb), kmin->data,
                                       kmax->data, static_cast<cudaStream_t>(stream));
  ++g_launches;
  return e == cudaSuccess ? FL_OK : cuda_fail(e, "rsa_summaries launch");
}

fl_status fl_rsa_build_summaries(const fl_tensor* k, fl_tensor* kmin, fl_tensor* kmax, int32_t blk_k, void* stream) {
  return rsa_summaries(k, kmin, kmax, blk_k, 0, stream);
}

fl_status fl_rsa_update_summaries(const fl_tensor* k, fl_tensor* kmin, fl_tensor* kmax, int32_t blk_k, int64_t k_begin,
                                  void* stream) {
  return rsa_summaries(k, kmin, kmax, blk_k, k_begin, stream);
}

fl_status fl_rsa_select(const fl_tensor* q, const fl_tensor* kmin, const fl_tensor* kmax, int32_t s_k, int32_t topk,
                        int32_t blk_q, int32_t blk_k, int32_t causal_align, fl_tensor* blk_idx, fl_tensor* blk_cnt,
                        void* stream) {
  if (!q || !kmin || !kmax || !blk_idx || !blk_cnt || !q->data || !kmin->data || !kmax->data || !blk_idx->data ||
      !blk_cnt->data)
    return fail(FL_ERR_INVALID_ARGUMENT, "rsa_select: q, kmin, kmax, blk_idx, blk_cnt are required");
  if (blk_q != 128 || blk_k != 128) return fail(FL_ERR_UNSUPPORTED, "rsa_select: blk_q == blk_k == 128");
  if (causal_align != 0 && causal_align != 1) return fail(FL_ERR_INVALID_ARGUMENT, "rsa_select: causal_align 0 or 1");
  if (q->dtype != FL_BF16 || kmin->dtype != FL_BF16 || kmax->dtype != FL_BF16)
    return fail(FL_ERR_UNSUPPORTED, "rsa_select: bf16 only");
  if (q->rank != 4 && q->rank != 5) return fail(FL_ERR_INVALID_ARGUMENT, "rsa_select: q rank 4 or 5");
  View5 qv;
  if (!to_view(*q, q->rank, 0, qv)) return fail(FL_ERR_SHAPE_MISMATCH, "rsa_select: bad q view");
  const int64_t B = qv.size[0], G = qv.size[1], Hq = qv.size[2], Sq = qv.size[3], D = qv.size[4];
  if (D != 64 && D != 128) return fail(FL_ERR_UNSUPPORTED, "rsa_select: D in {64, 128}");
  if (qv.stride[4] != 1) return fail(FL_ERR_UNSUPPORTED, "rsa_select: q last dim must be contiguous");
  if (s_k <= 0) return fail(FL_ERR_INVALID_ARGUMENT, "rsa_select: s_k must be > 0");
  const int64_t nkb = (s_k + blk_k - 1) / blk_k, nqb = (Sq + blk_q - 1) / blk_q;
  if (B * G == 0 || kmin->rank != 3 || kmin->size[0] % (B * G)) return fail(FL_ERR_SHAPE_MISMATCH, "rsa_select: kmin rank 3 [B*G*Hkv, n_kblk, D]");
  const int64_t Hkv = kmin->size[0] / (B * G);
  if (Hkv == 0 || Hq % Hkv) return fail(FL_ERR_SHAPE_MISMATCH, "rsa_select: Hq %% Hkv != 0");
  for (const fl_tensor* t : {kmin, kmax})
    if (t->rank != 3 || t->size[0] != B * G * Hkv || t->size[1] != nkb || t->size[2] != D || t->stride[2] != 1 ||
        t->stride[1] != D || t->stride[0] != nkb * D)
      return fail(FL_ERR_SHAPE_MISMATCH, "rsa_select: kmin/kmax must be contiguous [B*G*Hkv, ceil(s_k/blk_k), D]");
  if (topk < 0) return fail(FL_ERR_INVALID_ARGUMENT, "rsa_select: topk >= 0");
  const int64_t max_sel = blk_idx->size[2];
  if (blk_idx->dtype != FL_I32 || blk_cnt->dtype != FL_I32 || blk_idx->rank != 3 || blk_cnt->rank != 2 ||
      blk_idx->size[0] != B * G * Hq || blk_idx->size[1] != nqb || blk_idx->stride[2] != 1 ||
      blk_idx->stride[1] != max_sel || blk_idx->stride[0] != nqb * max_sel || blk_cnt->size[0] != B * G * Hq ||
      blk_cnt->size[1] != nqb || blk_cnt->stride[1] != 1 || blk_cnt->stride[0] != nqb)
    return fail(FL_ERR_SHAPE_MISMATCH, "rsa_select: blk_idx i32 [B*G*Hq, n_qblk, max_sel], blk_cnt i32 [B*G*Hq, n_qblk], contiguous");
  if (max_sel < topk + 2 || max_sel > 512) return fail(FL_ERR_INVALID_ARGUMENT, "rsa_select: topk + 2 <= max_sel <= 512");
  for (const void* ptr : {q->data, kmin->data, kmax->data, blk_idx->data, blk_cnt->data})
    if (!on_device(ptr)) return fail(FL_ERR_INVALID_ARGUMENT, "rsa_select: pointers must be device memory");
  if (Sq == 0 || Hq == 0) return FL_OK;
  RsaSelParams p{};
  p.B = (int)B; p.G = (int)G; p.Hq = (int)Hq; p.Hkv = (int)Hkv; p.grp = (int)(Hq / Hkv);
  p.Sq = (int)Sq; p.Sk = s_k; p.D = (int)D; p.nkb = (int)nkb; p.nqb = (int)nqb; p.topk = topk;
  p.max_sel = (int)max_sel; p.q_off = causal_align ? 0 : (int)(s_k - Sq);
  p.blk_idx = static_cast<int32_t*>(blk_idx->data); p.blk_cnt = static_cast<int32_t*>(blk_cnt->data);
  if (rsa_select_small_ok(p)) {                         // decode-sized query blocks: SIMT scores, one pass over summaries
    cudaError_t e = launch_rsa_select_small(p, qv.data, qv.size[0] > 1 ? qv.stride[0] : 0,
                                            qv.size[1] > 1 ? qv.stride[1] : 0, qv.size[2] > 1 ? qv.stride[2] : 0,
                                            qv.stride[3], kmin->data, kmax->data, static_cast<cudaStream_t>(stream));
    ++g_launches;
    return e == cudaSuccess ? FL_OK : cuda_fail(e, "rsa_select_small launch");
  }
  if (nkb > rsa_select_max_blocks((int)D))
    return fail(FL_ERR_UNSUPPORTED, "rsa_select: n_kblk %lld exceeds %d at D=%lld", (long long)nkb,
                rsa_select_max_blocks((int)D), (long long)D);
  CUtensorMap tq, tmn, tmx;
  int qbg, qbb, d0, d1;
  fl_status st;
  if ((st = encode_map(qv, 64, &tq, &qbg, &qbb)) != FL_OK) return st;
  for (int w = 0; w < 2; ++w) {
    const fl_tensor* t = w ? kmax : kmin;
    View5 sv;
    sv.present = true;
    sv.data = t->data;
    sv.dtype = FL_BF16;
    sv.size[2] = t->size[0]; sv.stride[2] = t->stride[0];
    sv.size[3] = t->size[1]; sv.stride[3] = t->stride[1];
    sv.size[4] = t->size[2]; sv.stride[4] = 1;
    if ((st = encode_map(sv, 64, w ? &tmx : &tmn, &d0, &d1)) != FL_OK) return st;
  }
  p.q_bcast_g = qbg; p.q_bcast_b = qbb;
  cudaError_t e = launch_rsa_select(p, tq, tmn, tmx, static_cast<cudaStream_t>(stream));
  ++g_launches;
  return e == cudaSuccess ? FL_OK : cuda_fail(e, "rsa_select launch");
}

const char* fl_status_string(fl_status s) {
  switch (s) {
    case FL_OK: return "FL_OK";
    case FL_ERR_INVALID_ARGUMENT: return "FL_ERR_INVALID_ARGUMENT";
    case FL_ERR_UNSUPPORTED: return "FL_ERR_UNSUPPORTED";
    case FL_ERR_MISALIGNED: return "FL_ERR_MISALIGNED";
    case FL_ERR_SHAPE_MISMATCH: return "FL_ERR_SHAPE_MISMATCH";
    case FL_ERR_WORKSPACE: return "FL_ERR_WORKSPACE";
    case FL_ERR_CUDA: return "FL_ERR_CUDA";
    case FL_ERR_ABI_VERSION: return "FL_ERR_ABI_VERSION";
  }
  return "FL_ERR_UNKNOWN";
}

size_t fl_attn_args_size(void) { return sizeof(fl_attn_args); }
size_t fl_attn_bwd_args_size(void) { return sizeof(fl_attn_bwd_args); }

fl_status fl_debug_timing(uint64_t* out48, int32_t reset) {
  if (!out48) return fail(FL_ERR_INVALID_ARGUMENT, "out48 is NULL");
  cudaError_t e = debug_timing(reinterpret_cast<unsigned long long*>(out48), reset);
  if (e == cudaErrorNotSupported) {
    cudaGetLastError();
    return fail(FL_ERR_UNSUPPORTED, "library built without -DFL_TIMING");
  }
  return e == cudaSuccess ? FL_OK : cuda_fail(e, "debug timing copy");
}

const char* fl_last_error(void) { return g_err.c_str(); }
int32_t fl_abi_version(void) { return FL_ABI_VERSION; }
int64_t fl_launch_count(int32_t reset) {
  int64_t n = g_launches;
  if (reset) g_launches = 0;
  return n;
}

}  // extern "C"
