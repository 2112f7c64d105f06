// toy.cu — the reference's toy transformer on the device around the attention kernels (SURVEY.md
// §8f rank 2; BASELINE configs[0]).
//
// Reference behaviour replaced: toy::ToyModel (toy_model.hpp:71-92, toy_model.cpp:45-221):
//   x = emb[id mod V]; per layer q, k, v = W x; interleaved RoPE per head at the token's Multiverse
//   position (toy_model.cpp:30-41); attention over the visible context then self (:121-157);
//   x += Wo attn; x += W_down tanh(W_up x); logits = unemb x.
// Here every piece runs on the GPU: the projections / MLP / unembed as fp32 tiled GEMMs (the
// reference is fp64; the parity bound is set by the bf16 attention inputs), RoPE in fp64 with the
// reference's own frequency expression, attention through K4 (mv_toy_step, one launch for all lanes,
// K/V appended into the paged store) or K3 (mv_toy_forward, masked prefill).
//
// Head dims 64 (C1: 4 heads x 64) and 128 run on the attention kernels' native head dims
// (mv_attn_head_dim).  Any other even head dim below 128 rides the 128-wide kernels zero-padded: zero
// q/k dims add nothing to q.k, zero v dims give zero outputs that are dropped, and q is pre-scaled by
// sqrt(128 / dh) so the kernels' 1/sqrt(128) becomes 1/sqrt(dh).  The rotation uses dh's frequencies,
// so q and k are rotated here and the kernels see position 0 (their identity rotation).
#include <cmath>
#include <cstring>
#include <vector>

#include "store.hpp"

struct mv_toy;

namespace mv {
namespace {

constexpr int kLinTile = 64, kLinK = 32;

// y[n][M] = x[n][K] . W[M][K]^T (MODE 0), y += (MODE 1), y = tanh(.) (MODE 2); fp32, one 64 x 64
// output tile per CTA, 4 x 4 per thread.
template <int MODE>
__global__ void __launch_bounds__(256) toy_linear_kernel(const float* __restrict__ x, const float* __restrict__ W,
                                                         float* __restrict__ y, int n, int M, int K) {
  __shared__ float xs[kLinTile][kLinK + 1], ws[kLinTile][kLinK + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int r0 = blockIdx.y * kLinTile, c0 = blockIdx.x * kLinTile;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += kLinK) {
    for (int e = threadIdx.x; e < kLinTile * kLinK; e += 256) {
      const int rr = e / kLinK, kk = e % kLinK;
      xs[rr][kk] = (r0 + rr < n && k0 + kk < K) ? x[(size_t)(r0 + rr) * K + k0 + kk] : 0.f;
      ws[rr][kk] = (c0 + rr < M && k0 + kk < K) ? W[(size_t)(c0 + rr) * K + k0 + kk] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < kLinK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = xs[ty * 4 + i][kk];
        b[i] = ws[tx * 4 + i][kk];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + ty * 4 + i;
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + tx * 4 + j;
      if (c >= M) continue;
      float* dst = y + (size_t)r * M + c;
      if (MODE == 0) *dst = acc[i][j];
      else if (MODE == 1) *dst += acc[i][j];
      else *dst = tanhf(acc[i][j]);
    }
  }
}

__global__ void toy_embed_kernel(const int32_t* __restrict__ tokens, int n, const float* __restrict__ emb, int V,
                                 int D, float* __restrict__ x) {
  const int i = blockIdx.x;
  if (i >= n) return;
  int id = tokens[i] % V;  // toy_model.cpp:97-98
  if (id < 0) id += V;
  for (int d = threadIdx.x; d < D; d += blockDim.x) x[(size_t)i * D + d] = emb[(size_t)id * D + d];
}

// qkv [n][3D] -> q, k, v bf16 [n][H][ad] (ad = attention head dim, zero-padded past dh), q and k rotated
// at pos with dh's frequencies (fp64 angle and sincos, toy_model.cpp:30-41), q scaled by sqrt(ad / dh).  Optionally the
// reference's cache record of the token for this layer: kv_rec[n][rec] at layer_off = [K (rotated) | V].
__global__ void toy_qkv_post_kernel(const float* __restrict__ qkv, const int32_t* __restrict__ pos, int n, int H,
                                    int dh, int ad, const double* __restrict__ inv, float qscale,
                                    __nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ k,
                                    __nv_bfloat16* __restrict__ v, float* __restrict__ kv_rec, int rec, int layer_off) {
  const int i = blockIdx.x;
  if (i >= n) return;
  const int D = H * dh;
  const float* row = qkv + (size_t)i * 3 * D;
  const int p = pos[i];
  for (int e = threadIdx.x; e < H * (ad / 2); e += blockDim.x) {  // (head, pair of the ad dims)
    const int h = e / (ad / 2), t = e % (ad / 2);
    const size_t o = ((size_t)i * H + h) * ad + 2 * t;
    if (2 * t >= dh) {
      q[o] = q[o + 1] = k[o] = k[o + 1] = v[o] = v[o + 1] = __float2bfloat16(0.f);
      continue;
    }
    double s, c;
    sincos((double)p * inv[t], &s, &c);
    const int d = h * dh + 2 * t;
    const double qa = row[d], qb = row[d + 1], ka = row[D + d], kb = row[D + d + 1];
    const float qr0 = (float)(qa * c - qb * s), qr1 = (float)(qa * s + qb * c);
    const float kr0 = (float)(ka * c - kb * s), kr1 = (float)(ka * s + kb * c);
    q[o] = __float2bfloat16(qr0 * qscale);
    q[o + 1] = __float2bfloat16(qr1 * qscale);
    k[o] = __float2bfloat16(kr0);
    k[o + 1] = __float2bfloat16(kr1);
    v[o] = __float2bfloat16(row[2 * D + d]);
    v[o + 1] = __float2bfloat16(row[2 * D + d + 1]);
    if (kv_rec) {
      float* r = kv_rec + (size_t)i * rec + layer_off;
      r[d] = kr0;
      r[d + 1] = kr1;
      r[D + d] = row[2 * D + d];
      r[D + d + 1] = row[2 * D + d + 1];
    }
  }
}

// attention output [n][H][ad] fp32 -> [n][D] (the first dh dims of each head)
__global__ void toy_gather_heads_kernel(const float* __restrict__ att, int n, int H, int dh, int ad,
                                        float* __restrict__ a) {
  const int i = blockIdx.x;
  if (i >= n) return;
  for (int e = threadIdx.x; e < H * dh; e += blockDim.x) a[(size_t)i * H * dh + e] = att[((size_t)i * H + e / dh) * ad + e % dh];
}

// reference cache records (fp64 [ctx][rec], per layer [K | V]) -> bf16 K, V [ctx][H][ad] of one layer
__global__ void toy_records_kernel(const double* __restrict__ recs, int n, int rec, int layer_off, int H, int dh,
                                   int ad, __nv_bfloat16* __restrict__ k, __nv_bfloat16* __restrict__ v) {
  const int i = blockIdx.x;
  if (i >= n) return;
  const int D = H * dh;
  for (int e = threadIdx.x; e < H * ad; e += blockDim.x) {
    const int h = e / ad, d = e % ad;
    const bool in = d < dh;
    k[(size_t)i * H * ad + e] = __float2bfloat16(in ? (float)recs[(size_t)i * rec + layer_off + h * dh + d] : 0.f);
    v[(size_t)i * H * ad + e] = __float2bfloat16(in ? (float)recs[(size_t)i * rec + layer_off + D + h * dh + d] : 0.f);
  }
}

__global__ void argmax_rows_kernel(const float* __restrict__ x, int n, int cols, int32_t* __restrict__ idx) {
  const int i = blockIdx.x;
  if (i >= n) return;
  float best = -INFINITY;
  int arg = 0;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    const float v = x[(size_t)i * cols + c];
    if (v > best) best = v, arg = c;  // first maximum within the thread's strided columns
  }
  __shared__ float sb[32];
  __shared__ int sa[32];
  for (int o = 16; o; o >>= 1) {
    const float ob = __shfl_down_sync(0xffffffffu, best, o);
    const int oa = __shfl_down_sync(0xffffffffu, arg, o);
    if (ob > best || (ob == best && oa < arg)) best = ob, arg = oa;
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) sb[w] = best, sa[w] = arg;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (sb[k] > best || (sb[k] == best && sa[k] < arg)) best = sb[k], arg = sa[k];
    idx[i] = arg;  // engine.cpp:543-556: the first index of the maximum
  }
}

template <int MODE>
void linear(const float* x, const float* W, float* y, int n, int M, int K, cudaStream_t st) {
  dim3 grid((M + kLinTile - 1) / kLinTile, (n + kLinTile - 1) / kLinTile);
  toy_linear_kernel<MODE><<<grid, 256, 0, st>>>(x, W, y, n, M, K);
}

}  // namespace

struct ToyDev {
  mv_toy_config cfg{};
  int D = 0, dh = 0, ad = 0, hidden = 0;  // ad: the attention kernels' head dim (mv_attn_head_dim(dh))
  float *emb = nullptr, *unemb = nullptr;
  std::vector<float*> wqkv, wo, up, down;  // per layer, device
  double* inv = nullptr;                   // [dh / 2] RoPE inverse frequencies
  // scratch (grown on demand)
  size_t cap_rows = 0;
  float *x = nullptr, *qkv = nullptr, *att = nullptr, *a = nullptr, *h = nullptr;
  __nv_bfloat16 *q = nullptr, *k = nullptr, *v = nullptr;
  int32_t* zero_pos = nullptr;
  void* ws = nullptr;
  size_t ws_bytes = 0;

  ~ToyDev() {
    cudaFree(emb);
    cudaFree(unemb);
    for (auto* p : wqkv) cudaFree(p);
    for (auto* p : wo) cudaFree(p);
    for (auto* p : up) cudaFree(p);
    for (auto* p : down) cudaFree(p);
    cudaFree(inv);
    free_scratch();
    cudaFree(ws);
  }
  void free_scratch() {
    for (void* p : {(void*)x, (void*)qkv, (void*)att, (void*)a, (void*)h, (void*)q, (void*)k, (void*)v, (void*)zero_pos})
      cudaFree(p);
    x = qkv = att = a = h = nullptr;
    q = k = v = nullptr;
    zero_pos = nullptr;
    cap_rows = 0;
  }
  mv_status ensure_rows(size_t n) {
    if (n <= cap_rows) return MV_OK;
    free_scratch();
    const size_t c = std::max<size_t>(n, 64);
    const int H = cfg.heads;
    MV_CUDA_TRY(cudaMalloc(&x, sizeof(float) * c * D));
    MV_CUDA_TRY(cudaMalloc(&qkv, sizeof(float) * c * 3 * D));
    MV_CUDA_TRY(cudaMalloc(&att, sizeof(float) * c * H * ad));
    MV_CUDA_TRY(cudaMalloc(&a, sizeof(float) * c * D));
    MV_CUDA_TRY(cudaMalloc(&h, sizeof(float) * c * hidden));
    MV_CUDA_TRY(cudaMalloc(&q, sizeof(__nv_bfloat16) * c * H * ad));
    MV_CUDA_TRY(cudaMalloc(&k, sizeof(__nv_bfloat16) * c * H * ad));
    MV_CUDA_TRY(cudaMalloc(&v, sizeof(__nv_bfloat16) * c * H * ad));
    MV_CUDA_TRY(cudaMalloc(&zero_pos, sizeof(int32_t) * c));
    MV_CUDA_TRY(cudaMemset(zero_pos, 0, sizeof(int32_t) * c));
    cap_rows = c;
    return MV_OK;
  }
  // post-attention half of a layer: x += Wo a; x += W_down tanh(W_up x)
  void finish_layer(int l, int n, cudaStream_t st) {
    toy_gather_heads_kernel<<<n, 128, 0, st>>>(att, n, cfg.heads, dh, ad, a);
    linear<1>(a, wo[l], x, n, D, D, st);
    linear<2>(x, up[l], h, n, hidden, D, st);
    linear<1>(h, down[l], x, n, D, hidden, st);
  }
};

}  // namespace mv

struct mv_toy {
  mv::ToyDev* impl;
};

using namespace mv;

extern "C" size_t mv_toy_weight_count(const mv_toy_config* c) {
  if (!c) return 0;
  const size_t D = (size_t)c->model_dim, V = (size_t)c->vocab, L = (size_t)c->layers;
  return 2 * V * D + L * (4 * D * D + 8 * D * D);
}

extern "C" mv_status mv_toy_create(const mv_toy_config* cfg, const double* h_weights, mv_toy** out) {
  if (!cfg || !h_weights || !out) return fail(MV_ERR_INVALID_ARGUMENT, "mv_toy_create: null argument");
  // toy_model.cpp:46-51
  if (cfg->layers < 1 || cfg->heads < 1 || cfg->model_dim < 1 || cfg->vocab < 1)
    return fail(MV_ERR_INVALID_ARGUMENT, "toy model dims must be >= 1");
  if (cfg->model_dim % cfg->heads != 0 || (cfg->model_dim / cfg->heads) % 2 != 0)
    return fail(MV_ERR_INVALID_ARGUMENT, "model_dim must split into even-sized heads");
  if (cfg->model_dim / cfg->heads > kHeadDim)
    return fail(MV_ERR_INVALID_ARGUMENT, "head_dim above the attention kernels' 128");
  auto* m = new ToyDev();
  m->cfg = *cfg;
  if (m->cfg.rope_base <= 0) m->cfg.rope_base = 10000.0;
  m->D = cfg->model_dim;
  m->dh = cfg->model_dim / cfg->heads;
  m->ad = mv_attn_head_dim(m->dh);
  m->hidden = 4 * cfg->model_dim;
  const size_t D = m->D, V = cfg->vocab, Hd = m->hidden;
  auto up32 = [&](const double* src, size_t count, float** dst) -> mv_status {
    std::vector<float> tmp(count);
    for (size_t i = 0; i < count; ++i) tmp[i] = (float)src[i];
    MV_CUDA_TRY(cudaMalloc(dst, sizeof(float) * count));
    MV_CUDA_TRY(cudaMemcpy(*dst, tmp.data(), sizeof(float) * count, cudaMemcpyHostToDevice));
    return MV_OK;
  };
  // ToyModelWeights order (toy_model.cpp:58-68): embedding, per layer wq wk wv wo w_up w_down, unembed
  const double* p = h_weights;
  mv_status st = up32(p, V * D, &m->emb);
  p += V * D;
  for (int l = 0; l < cfg->layers && st == MV_OK; ++l) {
    float* w = nullptr;
    st = up32(p, 3 * D * D, &w);  // wq, wk, wv are contiguous: one [3D][D] projection
    m->wqkv.push_back(w);
    p += 3 * D * D;
    if (st == MV_OK) st = up32(p, D * D, &w), m->wo.push_back(w);
    p += D * D;
    if (st == MV_OK) st = up32(p, Hd * D, &w), m->up.push_back(w);
    p += Hd * D;
    if (st == MV_OK) st = up32(p, D * Hd, &w), m->down.push_back(w);
    p += D * Hd;
  }
  if (st == MV_OK) st = up32(p, V * D, &m->unemb);
  if (st == MV_OK) {
    std::vector<double> inv(m->dh / 2);
    for (int t = 0; t < m->dh / 2; ++t) inv[t] = std::pow(m->cfg.rope_base, -2.0 * (double)t / (double)m->dh);
    if (cudaMalloc(&m->inv, sizeof(double) * inv.size()) != cudaSuccess ||
        cudaMemcpy(m->inv, inv.data(), sizeof(double) * inv.size(), cudaMemcpyHostToDevice) != cudaSuccess)
      st = fail(MV_ERR_CUDA, "mv_toy_create: RoPE table upload failed");
  }
  if (st != MV_OK) {
    delete m;
    return st;
  }
  *out = new mv_toy{m};
  return MV_OK;
}

extern "C" mv_status mv_toy_get_config(const mv_toy* m, mv_toy_config* out) {
  if (!m || !m->impl || !out) return fail(MV_ERR_INVALID_ARGUMENT, "null argument");
  *out = m->impl->cfg;
  return MV_OK;
}

extern "C" int32_t mv_toy_vocab(const mv_toy* m) { return m && m->impl ? m->impl->cfg.vocab : 0; }

extern "C" int32_t mv_attn_head_dim(int32_t model_head_dim) {
  return head_dim_supported(model_head_dim) ? model_head_dim : kHeadDim;
}

extern "C" mv_status mv_toy_destroy(mv_toy* m) {
  if (!m) return MV_OK;
  delete m->impl;
  delete m;
  return MV_OK;
}

static mv_status check_store(const ToyDev& m, mv_kv_store* s) {
  if (!s || !s->impl) return fail(MV_ERR_INVALID_ARGUMENT, "null store");
  const mv_kv_config& c = s->impl->cfg();
  if (c.kv_heads != m.cfg.heads || c.layers != m.cfg.layers || c.head_dim != m.ad)
    return fail(MV_ERR_INVALID_ARGUMENT,
                "store attention planes do not match the toy model (layers x heads x mv_attn_head_dim(d_h))");
  return MV_OK;
}

extern "C" mv_status mv_toy_step(mv_toy* tm, mv_kv_store* s, const uint64_t* h_handles, int32_t n,
                                 const int32_t* d_tokens, const int32_t* d_positions, float* d_logits,
                                 float* d_hidden, float* d_kv) {
  if (!tm || !tm->impl) return fail(MV_ERR_INVALID_ARGUMENT, "null toy model");
  ToyDev& m = *tm->impl;
  if (mv_status e = check_store(m, s)) return e;
  if (n <= 0) return n == 0 ? MV_OK : fail(MV_ERR_INVALID_ARGUMENT, "mv_toy_step: n < 0");
  if (!h_handles || !d_tokens || !d_positions || !d_logits) return fail(MV_ERR_INVALID_ARGUMENT, "null buffer");
  PagedStore& st = *s->impl;
  cudaStream_t cs = st.stream();
  if (mv_status e = m.ensure_rows(n)) return e;
  const int H = m.cfg.heads, D = m.D, L = m.cfg.layers, rec = 2 * L * D;
  const float qscale = sqrtf((float)m.ad / (float)m.dh);
  toy_embed_kernel<<<n, 128, 0, cs>>>(d_tokens, n, m.emb, m.cfg.vocab, D, m.x);
  MV_LAUNCH_CHECK();
  for (int l = 0; l < L; ++l) {
    linear<0>(m.x, m.wqkv[l], m.qkv, n, 3 * D, D, cs);
    toy_qkv_post_kernel<<<n, 128, 0, cs>>>(m.qkv, d_positions, n, H, m.dh, m.ad, m.inv, qscale, m.q, m.k, m.v, d_kv, rec,
                                            l * 2 * D);
    MV_LAUNCH_CHECK();
    // engine.cpp:639-641 (extend + release) in place: the token joins each lane's cache, K already
    // rotated (position 0 = identity in the kernels)
    mv_status e = l == 0 ? st.append(h_handles, n, d_tokens, m.zero_pos, 0, m.k, m.v)
                         : st.write_last(h_handles, n, m.zero_pos, l, m.k, m.v);
    if (e) return e;
    if ((e = mv_attn_decode(s, l, h_handles, n, H, m.q, m.zero_pos, m.att, 1))) return e;
    m.finish_layer(l, n, cs);
    MV_LAUNCH_CHECK();
  }
  if (d_hidden) MV_CUDA_TRY(cudaMemcpyAsync(d_hidden, m.x, sizeof(float) * n * D, cudaMemcpyDeviceToDevice, cs));
  linear<0>(m.x, m.unemb, d_logits, n, m.cfg.vocab, D, cs);
  MV_LAUNCH_CHECK();
  return MV_OK;
}

extern "C" mv_status mv_toy_load_context(mv_toy* tm, mv_kv_store* s, uint64_t h, const double* h_records,
                                         int64_t ctx_len) {
  if (!tm || !tm->impl) return fail(MV_ERR_INVALID_ARGUMENT, "null toy model");
  ToyDev& m = *tm->impl;
  if (mv_status e = check_store(m, s)) return e;
  if (ctx_len < 0 || (ctx_len > 0 && !h_records)) return fail(MV_ERR_INVALID_ARGUMENT, "mv_toy_load_context: bad context");
  if (ctx_len == 0) return MV_OK;
  PagedStore& st = *s->impl;
  cudaStream_t cs = st.stream();
  if (mv_status e = m.ensure_rows(ctx_len)) return e;
  const int H = m.cfg.heads, D = m.D, L = m.cfg.layers, rec = 2 * L * D;
  double* d_rec = nullptr;
  MV_CUDA_TRY(cudaMallocAsync(&d_rec, sizeof(double) * ctx_len * rec, cs));
  MV_CUDA_TRY(cudaMemcpyAsync(d_rec, h_records, sizeof(double) * ctx_len * rec, cudaMemcpyHostToDevice, cs));
  int64_t base = 0;
  if (mv_status e = st.length(h, &base)) return e;
  for (int l = 0; l < L; ++l) {
    toy_records_kernel<<<(unsigned)ctx_len, 128, 0, cs>>>(d_rec, (int)ctx_len, rec, l * 2 * D, H, m.dh, m.ad, m.k, m.v);
    MV_LAUNCH_CHECK();
    // the records hold post-RoPE K: positions 0 (identity) for the store's rotation
    mv_status e = l == 0 ? st.append_many(h, ctx_len, nullptr, m.zero_pos, 0, m.k, m.v)
                         : st.write_range(h, base, ctx_len, m.zero_pos, l, m.k, m.v);
    if (e) return e;
  }
  MV_CUDA_TRY(cudaFreeAsync(d_rec, cs));
  return MV_OK;
}

extern "C" mv_status mv_toy_forward(mv_toy* tm, const int32_t* d_tokens, int32_t n, const int32_t* d_positions,
                                    const int32_t* d_excl, int32_t max_depth, float* d_logits, float* d_hidden,
                                    mv_stream_t stream) {
  if (!tm || !tm->impl) return fail(MV_ERR_INVALID_ARGUMENT, "null toy model");
  if (n <= 0) return n == 0 ? MV_OK : fail(MV_ERR_INVALID_ARGUMENT, "mv_toy_forward: n < 0");
  if (!d_tokens || !d_positions || !d_excl || !d_logits) return fail(MV_ERR_INVALID_ARGUMENT, "null buffer");
  ToyDev& m = *tm->impl;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (mv_status e = m.ensure_rows(n)) return e;
  const int H = m.cfg.heads, D = m.D, L = m.cfg.layers;
  const size_t ws = mv_prefill_workspace_size_hd(n, H, H, m.ad);
  if (ws > m.ws_bytes) {
    cudaFree(m.ws);
    m.ws = nullptr;
    MV_CUDA_TRY(cudaMalloc(&m.ws, ws));
    m.ws_bytes = ws;
  }
  const float qscale = sqrtf((float)m.ad / (float)m.dh);
  toy_embed_kernel<<<n, 128, 0, cs>>>(d_tokens, n, m.emb, m.cfg.vocab, D, m.x);
  MV_LAUNCH_CHECK();
  for (int l = 0; l < L; ++l) {
    linear<0>(m.x, m.wqkv[l], m.qkv, n, 3 * D, D, cs);
    toy_qkv_post_kernel<<<n, 128, 0, cs>>>(m.qkv, d_positions, n, H, m.dh, m.ad, m.inv, qscale, m.q, m.k, m.v, nullptr, 0,
                                            0);
    MV_LAUNCH_CHECK();
    // ToyModel::forward (toy_model.cpp:174-202): every row over its mask-visible rows, then self
    if (mv_status e = mv_attn_prefill_hd(m.q, m.k, m.v, m.zero_pos, d_excl, max_depth, n, H, H, m.ad, m.cfg.rope_base,
                                         m.att, 1, m.ws, m.ws_bytes, stream))
      return e;
    m.finish_layer(l, n, cs);
    MV_LAUNCH_CHECK();
  }
  if (d_hidden) MV_CUDA_TRY(cudaMemcpyAsync(d_hidden, m.x, sizeof(float) * n * D, cudaMemcpyDeviceToDevice, cs));
  linear<0>(m.x, m.unemb, d_logits, n, m.cfg.vocab, D, cs);
  MV_LAUNCH_CHECK();
  return MV_OK;
}

extern "C" mv_status mv_argmax_rows(const float* d_x, int32_t n, int32_t cols, int32_t* d_idx, mv_stream_t stream) {
  if (n < 0 || cols <= 0 || (n > 0 && (!d_x || !d_idx))) return fail(MV_ERR_INVALID_ARGUMENT, "mv_argmax_rows: bad arguments");
  if (n == 0) return MV_OK;
  argmax_rows_kernel<<<n, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(d_x, n, cols, d_idx);
  MV_LAUNCH_CHECK();
  return MV_OK;
}
