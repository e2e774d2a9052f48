// Llama-shape stage compute: bf16 weights in HBM, fp32 residual stream.
//
// Per layer (reference layer_step structure, `/root/reference/pkg/src/treepipe/
// model.py:250-280`, with the Llama block: RMSNorm, RoPE, GQA, SwiGLU):
//
//   QKV  = Xd . Wqkv^T      K2 (epilogue: RoPE(q,k); q -> Xq; k,v -> KV rows in place)
//   attn = tree-attention(Xq, KV, ancestor bits)      K1 (attn.cu)      -> Xo
//   x   += Xo . Wo^T        K2 (epilogue: residual add)
//   Xd   = rmsnorm(x)
//   Xf   = silu(G) * U      K2 over the gate/up weights (64-row interleave; epilogue: SwiGLU)
//   x   += Xf . Wdown^T     K2 (epilogue: residual add)
//   Xd   = rmsnorm(x)                                   (input of the next layer)
//
// 9 launches per layer; every GEMM is a programmatic-dependent launch whose
// weight prologue overlaps the preceding kernel.
//
// Numerics (mirrored by oracle/llama.py): GEMM inputs bf16, accumulation and
// residual fp32; RoPE (HF rotate-half, angle in fp64) on the fp32 GEMM
// output, then rounded to bf16 for the cache / attention; softmax fp32.
#include <cmath>
#include <cstring>

#include "attn.h"
#include "gemm_tc.h"
#include "internal.h"

namespace tp {

enum { kCtrQkv = 0, kCtrO, kCtrGu, kCtrDown, kCtrHead, kCtrKinds };

struct LlamaModelExt {
  std::vector<CUtensorMap> qkv, o, gu, down;
  CUtensorMap head;
};

struct LlamaStageExt {
  int np = 0;  // padded node rows (multiple of 16)
  __nv_bfloat16 *Xd = nullptr, *Xo = nullptr, *Xf = nullptr, *Xq = nullptr;
  __nv_bfloat16 *kself = nullptr, *vself = nullptr;
  float* part = nullptr;
  size_t part_floats = 0;
  int* counters = nullptr;  // [kCtrKinds][ctr_stride]
  int ctr_stride = 0;
  float* rope = nullptr;  // [np][64][2]
  CUtensorMap mXd, mXo, mXf;
  float *pm = nullptr, *pl = nullptr, *po = nullptr;
  int max_chunks = 0;
};

static LlamaModelExt* mext(tp_model* m) { return reinterpret_cast<LlamaModelExt*>(m->tma_cache); }
static LlamaStageExt* sext(tp_stage* s) { return reinterpret_cast<LlamaStageExt*>(s->ext); }

// ---- kernels --------------------------------------------------------------------

__global__ void llama_embed_kernel(const __nv_bfloat16* __restrict__ E, const int32_t* __restrict__ tok, int d,
                                   float* __restrict__ x) {
  const int c = blockIdx.x;
  const __nv_bfloat16* e = E + (size_t)tok[c] * d;
  for (int j = threadIdx.x; j < d; j += blockDim.x) x[(size_t)c * d + j] = __bfloat162float(e[j]);
}

constexpr int kNormThreads = 1024;
constexpr int kNormPer = 8;  // d <= 8192

__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum_f32(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    float t = l < nw ? red[l] : 0.f;
    t = warp_sum_f32(t);
    if (l == 0) red[32] = t;
  }
  __syncthreads();
  const float t = red[32];
  __syncthreads();
  return t;
}

// Xd[c] = bf16(x[c] * 1/sqrt(mean(x[c]^2) + eps)); one CTA per node row, the
// same reduction shape at every call site (stage boundaries included).
__global__ void __launch_bounds__(kNormThreads) rmsnorm_kernel(const float* __restrict__ x, int d, float eps,
                                                               __nv_bfloat16* __restrict__ xd) {
  pdl_trigger();  // the following GEMM may start streaming its weights
  __shared__ float red[33];
  const float* xr = x + (size_t)blockIdx.x * d;
  float v[kNormPer];
  float ss = 0.f;
#pragma unroll
  for (int u = 0; u < kNormPer; ++u) {
    const int j = threadIdx.x + u * kNormThreads;
    v[u] = j < d ? xr[j] : 0.f;
  }
#pragma unroll
  for (int u = 0; u < kNormPer; ++u) {
    const int j = threadIdx.x + u * kNormThreads;
    if (j < d) ss += v[u] * v[u];
  }
  ss = block_sum(ss, red);
  const float r = 1.0f / sqrtf(ss / (float)d + eps);
#pragma unroll
  for (int u = 0; u < kNormPer; ++u) {
    const int j = threadIdx.x + u * kNormThreads;
    if (j < d) xd[(size_t)blockIdx.x * d + j] = __float2bfloat16_rn(v[u] * r);
  }
}

// cos/sin of every (node position, rotary pair) for the QKV epilogue; angle in fp64.
__global__ void rope_table_kernel(const int32_t* __restrict__ pos, double theta, float* __restrict__ out) {
  const int c = blockIdx.x, i = threadIdx.x;  // i in [0, 64)
  const double inv = pow(theta, -2.0 * (double)i / 128.0);
  double sn, cs;
  sincos((double)pos[c] * inv, &sn, &cs);
  out[((size_t)c * 64 + i) * 2] = (float)cs;
  out[((size_t)c * 64 + i) * 2 + 1] = (float)sn;
}

// ---- host ---------------------------------------------------------------------------

static int build_model_ext(tp_model* m) {
  if (m->tma_cache) return TP_OK;
  const tp_model_config& c = m->cfg;
  const int64_t d = c.hidden, q = (int64_t)c.heads * 128, kv = (int64_t)c.kv_heads * 128, f = c.ffn;
  auto* e = new LlamaModelExt();
  for (int l = c.layer_lo; l < c.layer_hi; ++l) {
    const tp_layer_weights& w = m->layers[l - c.layer_lo];
    CUtensorMap a, b, g, dn;
    TP_TRY(make_tmap_kmajor(&a, w.w[1], q + 2 * kv, d, 128));
    TP_TRY(make_tmap_kmajor(&b, w.w[4], d, q, 128));
    TP_TRY(make_tmap_kmajor(&g, w.w[5], 2 * f, d, 128));
    TP_TRY(make_tmap_kmajor(&dn, w.w[7], d, f, 128));
    e->qkv.push_back(a);
    e->o.push_back(b);
    e->gu.push_back(g);
    e->down.push_back(dn);
  }
  if (m->head) TP_TRY(make_tmap_kmajor(&e->head, m->head, c.vocab, d, 128));
  m->tma_cache = e;
  return TP_OK;
}

void llama_model_free(tp_model* m) {
  delete mext(m);
  m->tma_cache = nullptr;
}

int llama_workspace_bytes(const tp_model*, int, size_t* bytes) {
  *bytes = 256;  // llama state lives in LlamaStageExt
  return TP_OK;
}

int llama_init_weights(tp_model* m, uint64_t seed, cudaStream_t st) {
  const tp_model_config& c = m->cfg;
  const int64_t V = c.vocab, d = c.hidden, q = (int64_t)c.heads * 128, kv = (int64_t)c.kv_heads * 128, f = c.ffn;
  const int64_t per_layer = d * q + 2 * d * kv + q * d + 3 * d * f;
  auto sc = [&](int64_t fan_in) { return c.weight_scale ? std::sqrt(3.0 / (double)fan_in) / 0.1 : 1.0; };
  if (m->embed) TP_TRY(lcg_fill_bf16((__nv_bfloat16*)m->embed, V * d, seed, 0, 1.0, st));
  for (int l = c.layer_lo; l < c.layer_hi; ++l) {
    const tp_layer_weights& w = m->layers[l - c.layer_lo];
    int64_t off = V * d + (int64_t)l * per_layer;
    auto* qkv = (__nv_bfloat16*)w.w[1];
    TP_TRY(lcg_fill_bf16_rows(qkv, d, q, seed, off, sc(d), 0, 0, st));  // Wq [d, q]
    off += d * q;
    TP_TRY(lcg_fill_bf16_rows(qkv, d, kv, seed, off, sc(d), q, 0, st));  // Wk
    off += d * kv;
    TP_TRY(lcg_fill_bf16_rows(qkv, d, kv, seed, off, sc(d), q + kv, 0, st));  // Wv
    off += d * kv;
    TP_TRY(lcg_fill_bf16_rows((__nv_bfloat16*)w.w[4], q, d, seed, off, sc(q), 0, 0, st));  // Wo [q, d]
    off += q * d;
    TP_TRY(lcg_fill_bf16_rows((__nv_bfloat16*)w.w[5], d, f, seed, off, sc(d), 0, 1, st));  // Wgate
    off += d * f;
    TP_TRY(lcg_fill_bf16_rows((__nv_bfloat16*)w.w[5], d, f, seed, off, sc(d), 64, 1, st));  // Wup
    off += d * f;
    TP_TRY(lcg_fill_bf16_rows((__nv_bfloat16*)w.w[7], f, d, seed, off, sc(f), 0, 0, st));  // Wdown [f, d]
  }
  if (m->head)
    TP_TRY(lcg_fill_bf16_rows((__nv_bfloat16*)m->head, d, V, seed, V * d + (int64_t)c.layers * per_layer, sc(d),
                              0, 0, st));
  TP_CUDA(cudaStreamSynchronize(st));
  return build_model_ext(m);
}

int llama_stage_init(tp_stage* s) {
  tp_model* m = s->m;
  const tp_model_config& c = m->cfg;
  TP_TRY(build_model_ext(m));
  LlamaStageExt* e = sext(s);
  if (e == nullptr) {
    e = new LlamaStageExt();
    s->ext = e;
    const int64_t d = c.hidden, q = (int64_t)c.heads * 128, kv = (int64_t)c.kv_heads * 128, f = c.ffn;
    e->np = (c.max_nodes + 15) / 16 * 16;
    const int64_t np = e->np;
    TP_CUDA(cudaMalloc(&e->Xd, np * d * 2));
    TP_CUDA(cudaMalloc(&e->Xo, np * q * 2));
    TP_CUDA(cudaMalloc(&e->Xf, np * f * 2));
    TP_CUDA(cudaMalloc(&e->Xq, np * q * 2));
    TP_CUDA(cudaMalloc(&e->kself, np * kv * 2));
    TP_CUDA(cudaMalloc(&e->vself, np * kv * 2));
    TP_CUDA(cudaMalloc(&e->rope, np * 64 * 2 * 4));
    TP_CUDA(cudaMemset(e->Xd, 0, np * d * 2));
    TP_CUDA(cudaMemset(e->Xo, 0, np * q * 2));
    TP_CUDA(cudaMemset(e->Xf, 0, np * f * 2));
    size_t pf = 0;
    int mt = 1;
    const int nmax = c.max_nodes;
    for (SkPlan p : {sk_plan((int)(q + 2 * kv), (int)d, nmax), sk_plan((int)d, (int)q, nmax),
                     sk_plan((int)(2 * f), (int)d, nmax), sk_plan((int)d, (int)f, nmax)}) {
      pf = std::max(pf, sk_part_floats(p));
      mt = std::max(mt, p.mtiles);
    }
    if (m->head) {
      SkPlan ph = sk_plan(c.vocab, (int)d, nmax);
      pf = std::max(pf, sk_part_floats(ph));
      mt = std::max(mt, ph.mtiles);
    }
    e->part_floats = pf;
    TP_CUDA(cudaMalloc(&e->part, pf * 4));
    e->ctr_stride = 2 * mt;  // arrivals | reducers done, per GEMM kind
    TP_CUDA(cudaMalloc(&e->counters, (size_t)kCtrKinds * e->ctr_stride * 4));
    TP_CUDA(cudaMemset(e->counters, 0, (size_t)kCtrKinds * e->ctr_stride * 4));
    TP_TRY(make_tmap_kmajor(&e->mXd, e->Xd, np, d, 16));
    TP_TRY(make_tmap_kmajor(&e->mXo, e->Xo, np, q, 16));
    TP_TRY(make_tmap_kmajor(&e->mXf, e->Xf, np, f, 16));
  }
  // attention chunk partials follow the KV capacity (+ ancestors + self)
  const int chunks = (s->cap + kAttnMaxExtra + 1 + kAttnChunk - 1) / kAttnChunk;
  if (chunks > e->max_chunks) {
    if (e->pm) cudaFree(e->pm);
    if (e->pl) cudaFree(e->pl);
    if (e->po) cudaFree(e->po);
    const size_t cells = (size_t)e->np * c.heads * chunks;
    TP_CUDA(cudaMalloc(&e->pm, cells * 4));
    TP_CUDA(cudaMalloc(&e->pl, cells * 4));
    TP_CUDA(cudaMalloc(&e->po, cells * 128 * 4));
    e->max_chunks = chunks;
  }
  return TP_OK;
}

void llama_stage_free(tp_stage* s) {
  LlamaStageExt* e = sext(s);
  if (!e) return;
  for (void* p : {(void*)e->Xd, (void*)e->Xo, (void*)e->Xf, (void*)e->Xq, (void*)e->kself, (void*)e->vself,
                  (void*)e->part, (void*)e->counters, (void*)e->rope, (void*)e->pm, (void*)e->pl, (void*)e->po})
    if (p) cudaFree(p);
  delete e;
  s->ext = nullptr;
}

int llama_embed(tp_model* m, int n, const int32_t* d_tokens, float* out, cudaStream_t st) {
  TP_CHECK(m->embed, TP_ECONFIG, "model has no embedding table");
  ::tp::count_launch(), llama_embed_kernel<<<n, 256, 0, st>>>((const __nv_bfloat16*)m->embed, d_tokens,
                                                              m->cfg.hidden, out);
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

static GemmEpi epi_base(LlamaStageExt* e, int kind) {
  GemmEpi g;
  g.part = e->part;
  g.counters = e->counters + (size_t)kind * e->ctr_stride;
  return g;
}

int llama_logits(tp_model* m, tp_stage* ws, int n, const float* x, float* logits, cudaStream_t st) {
  TP_CHECK(m->head, TP_ECONFIG, "model has no LM head");
  TP_TRY(llama_stage_init(ws));
  LlamaStageExt* e = sext(ws);
  const int d = m->cfg.hidden, V = m->cfg.vocab;
  ::tp::count_launch(), rmsnorm_kernel<<<n, kNormThreads, 0, st>>>(x, d, m->cfg.norm_eps, e->Xd);
  TP_CUDA(cudaGetLastError());
  GemmEpi g = epi_base(e, kCtrHead);
  g.op = kOpStore;
  g.out = logits;
  g.out_ld = V;
  return sk_gemm(&mext(m)->head, &e->mXd, sk_plan(V, d, n), g, st);
}

int llama_forward(tp_stage* s, const LevelDev& lv, const void* hidden_in, void* hidden_out, cudaStream_t st) {
  tp_model* m = s->m;
  const tp_model_config& c = m->cfg;
  TP_TRY(llama_stage_init(s));
  LlamaStageExt* e = sext(s);
  LlamaModelExt* me = mext(m);
  const int n = lv.n, d = c.hidden, H = c.heads, KV = c.kv_heads, f = c.ffn;
  const int q = H * 128, kvd = KV * 128;
  float* x = (float*)hidden_out;
  if (hidden_in) {
    if (hidden_in != hidden_out)
      TP_CUDA(cudaMemcpyAsync(x, hidden_in, (size_t)n * d * 4, cudaMemcpyDeviceToDevice, st));
  } else {
    TP_TRY(llama_embed(m, n, lv.tokens, x, st));
  }
  if (lv.layer_lo == lv.layer_hi) return TP_OK;
  ::tp::count_launch(), rope_table_kernel<<<n, 64, 0, st>>>(lv.positions, (double)c.rope_theta, e->rope);
  TP_CUDA(cudaGetLastError());
  ::tp::count_launch(), rmsnorm_kernel<<<n, kNormThreads, 0, st>>>(x, d, c.norm_eps, e->Xd);
  TP_CUDA(cudaGetLastError());
  const SkPlan pqkv = sk_plan(q + 2 * kvd, d, n), po = sk_plan(d, q, n), pgu = sk_plan(2 * f, d, n),
               pdn = sk_plan(d, f, n);
  AttnArgs aa;
  aa.q = e->Xq;
  aa.q_stride = q;
  aa.cap = s->cap;
  aa.kself = lv.append ? nullptr : e->kself;
  aa.vself = lv.append ? nullptr : e->vself;
  aa.H = H;
  aa.KV = KV;
  aa.scale = (float)(1.0 / std::sqrt(128.0));
  aa.pm = e->pm;
  aa.pl = e->pl;
  aa.po = e->po;
  aa.max_chunks = e->max_chunks;
  aa.out = e->Xo;
  aa.out_stride = q;
  GemmEpi gq = epi_base(e, kCtrQkv);
  gq.op = kOpQkv;
  gq.H = H;
  gq.KV = KV;
  gq.cap = s->cap;
  gq.row0 = lv.row0;
  gq.append = lv.append;
  gq.rope = e->rope;
  gq.xq = e->Xq;
  gq.kself = e->kself;
  gq.vself = e->vself;
  GemmEpi gr = epi_base(e, kCtrO);
  gr.op = kOpResid;
  gr.out = x;
  gr.out_ld = d;
  GemmEpi gd = gr;
  gd.counters = e->counters + (size_t)kCtrDown * e->ctr_stride;
  GemmEpi gg = epi_base(e, kCtrGu);
  gg.op = kOpSwiglu;
  gg.xf = e->Xf;
  gg.f = f;
  for (int layer = lv.layer_lo; layer < lv.layer_hi; ++layer) {
    const int li = layer - c.layer_lo;
    gq.kc = (__nv_bfloat16*)s->k[layer - s->lo];
    gq.vc = (__nv_bfloat16*)s->v[layer - s->lo];
    TP_TRY(sk_gemm(&me->qkv[li], &e->mXd, pqkv, gq, st));
    aa.k = gq.kc;
    aa.v = gq.vc;
    TP_TRY(attn_tree(aa, lv, st));
    TP_TRY(sk_gemm(&me->o[li], &e->mXo, po, gr, st));
    ::tp::count_launch(), rmsnorm_kernel<<<n, kNormThreads, 0, st>>>(x, d, c.norm_eps, e->Xd);
    TP_CUDA(cudaGetLastError());
    TP_TRY(sk_gemm(&me->gu[li], &e->mXd, pgu, gg, st));
    TP_TRY(sk_gemm(&me->down[li], &e->mXf, pdn, gd, st));
    if (layer + 1 < lv.layer_hi) {
      ::tp::count_launch(), rmsnorm_kernel<<<n, kNormThreads, 0, st>>>(x, d, c.norm_eps, e->Xd);
      TP_CUDA(cudaGetLastError());
    }
  }
  return TP_OK;
}

}  // namespace tp
