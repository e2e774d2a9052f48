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

// Grouped rmsnorm: one CTA per (node row, member).
struct NormGroup {
  const float* x[kMaxGroup];
  __nv_bfloat16* xd[kMaxGroup];
  int n[kMaxGroup];
};

__global__ void __launch_bounds__(kNormThreads) rmsnorm_group_kernel(const __grid_constant__ NormGroup ng, int d,
                                                                     float eps) {
  pdl_trigger();
  const int g = blockIdx.y;
  if ((int)blockIdx.x >= ng.n[g]) return;
  __shared__ float red[33];
  const float* xr = ng.x[g] + (size_t)blockIdx.x * d;
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
  __nv_bfloat16* out = ng.xd[g] + (size_t)blockIdx.x * d;
#pragma unroll
  for (int u = 0; u < kNormPer; ++u) {
    const int j = threadIdx.x + u * kNormThreads;
    if (j < d) out[j] = __float2bfloat16_rn(v[u] * r);
  }
}

int llama_forward(tp_stage* s, const LevelDev& lv, const void* hidden_in, void* hidden_out, cudaStream_t st) {
  tp_stage* ss[1] = {s};
  const void* hin[1] = {hidden_in};
  void* hout[1] = {hidden_out};
  return llama_forward_group(ss, &lv, hin, hout, 1, st);
}

// Several stages' levels on one device, layer slot by layer slot: slot j runs
// layer lo_g + j of every member g that has one, each GEMM as ONE grouped
// launch over the members (same segment boundaries as ungrouped launches, so
// every member's bits equal its stand-alone forward).
int llama_forward_group(tp_stage* const* ss, const LevelDev* lvs, const void* const* hin, void* const* hout,
                        int count, cudaStream_t st) {
  TP_CHECK(count >= 1 && count <= kMaxGroup, TP_ECONFIG, "stage group size outside [1, 8]");
  tp_model* m0 = ss[0]->m;
  const tp_model_config& c = m0->cfg;
  const int d = c.hidden, H = c.heads, KV = c.kv_heads, f = c.ffn;
  const int q = H * 128, kvd = KV * 128;
  int slots = 0;
  for (int g = 0; g < count; ++g) {
    tp_stage* s = ss[g];
    const tp_model_config& cg = s->m->cfg;
    TP_CHECK(cg.hidden == d && cg.heads == H && cg.kv_heads == KV && cg.ffn == f && cg.device == c.device,
             TP_ECONFIG, "grouped stages must share the model shape and device");
    TP_TRY(llama_stage_init(s));
    const LevelDev& lv = lvs[g];
    float* x = (float*)hout[g];
    if (hin[g]) {
      if (hin[g] != hout[g])
        TP_CUDA(cudaMemcpyAsync(x, hin[g], (size_t)lv.n * d * 4, cudaMemcpyDeviceToDevice, st));
    } else {
      TP_TRY(llama_embed(s->m, lv.n, lv.tokens, x, st));
    }
    slots = std::max(slots, lv.layer_hi - lv.layer_lo);
  }
  if (slots == 0) return TP_OK;
  int maxn = 0;
  for (int g = 0; g < count; ++g) {
    const LevelDev& lv = lvs[g];
    if (lv.layer_hi == lv.layer_lo) continue;
    maxn = std::max(maxn, lv.n);
    ::tp::count_launch(), rope_table_kernel<<<lv.n, 64, 0, st>>>(lv.positions, (double)c.rope_theta,
                                                                  sext(ss[g])->rope);
    TP_CUDA(cudaGetLastError());
  }
  const SkPlan pqkv = sk_plan(q + 2 * kvd, d, 1), po = sk_plan(d, q, 1), pgu = sk_plan(2 * f, d, 1),
               pdn = sk_plan(d, f, 1);
  for (int j = 0; j < slots; ++j) {
    int idx[kMaxGroup], na = 0;
    for (int g = 0; g < count; ++g)
      if (lvs[g].layer_lo + j < lvs[g].layer_hi) idx[na++] = g;
    NormGroup ng;
    GemmGroup gq, go, ggu, gdn;
    gq.count = go.count = ggu.count = gdn.count = na;
    int mx = 16;
    for (int a = 0; a < na; ++a) {
      const int g = idx[a];
      tp_stage* s = ss[g];
      const LevelDev& lv = lvs[g];
      LlamaStageExt* e = sext(s);
      LlamaModelExt* me = mext(s->m);
      const int layer = lv.layer_lo + j, li = layer - s->m->cfg.layer_lo;
      const int n = lv.n, npad = std::max(16, (n + 15) / 16 * 16);
      mx = std::max(mx, npad);
      float* x = (float*)hout[g];
      ng.x[a] = x;
      ng.xd[a] = e->Xd;
      ng.n[a] = n;
      GemmEpi eq = epi_base(e, kCtrQkv);
      eq.op = kOpQkv;
      eq.H = H;
      eq.KV = KV;
      eq.cap = s->cap;
      eq.row0 = lv.row0;
      eq.append = lv.append;
      eq.rope = e->rope;
      eq.xq = e->Xq;
      eq.kself = e->kself;
      eq.vself = e->vself;
      eq.kc = (__nv_bfloat16*)s->k[layer - s->lo];
      eq.vc = (__nv_bfloat16*)s->v[layer - s->lo];
      GemmEpi er = epi_base(e, kCtrO);
      er.op = kOpResid;
      er.out = x;
      er.out_ld = d;
      GemmEpi ed = er;
      ed.counters = e->counters + (size_t)kCtrDown * e->ctr_stride;
      GemmEpi eg = epi_base(e, kCtrGu);
      eg.op = kOpSwiglu;
      eg.xf = e->Xf;
      eg.f = f;
      auto set = [&](GemmGroup& gg, const CUtensorMap& wa, const CUtensorMap& xb, const GemmEpi& ep) {
        gg.m[a].a = wa;
        gg.m[a].b = xb;
        gg.m[a].e = ep;
        gg.m[a].n = n;
        gg.m[a].n_pad = npad;
      };
      set(gq, me->qkv[li], e->mXd, eq);
      set(go, me->o[li], e->mXo, er);
      set(ggu, me->gu[li], e->mXd, eg);
      set(gdn, me->down[li], e->mXf, ed);
    }
    gq.max_npad = go.max_npad = ggu.max_npad = gdn.max_npad = mx;
    if (j == 0) {
      ::tp::count_launch(), rmsnorm_group_kernel<<<dim3(maxn, na), kNormThreads, 0, st>>>(ng, d, c.norm_eps);
      TP_CUDA(cudaGetLastError());
    }
    TP_TRY(sk_gemm_group(gq, pqkv, st));
    AttnArgs aa[kMaxGroup];
    LevelDev al[kMaxGroup];
    for (int a = 0; a < na; ++a) {
      const int g = idx[a];
      tp_stage* s = ss[g];
      const LevelDev& lv = lvs[g];
      LlamaStageExt* e = sext(s);
      AttnArgs& x = aa[a];
      x.q = e->Xq;
      x.q_stride = q;
      x.cap = s->cap;
      x.kself = lv.append ? nullptr : e->kself;
      x.vself = lv.append ? nullptr : e->vself;
      x.H = H;
      x.KV = KV;
      x.scale = (float)(1.0 / std::sqrt(128.0));
      x.pm = e->pm;
      x.pl = e->pl;
      x.po = e->po;
      x.max_chunks = e->max_chunks;
      x.out = e->Xo;
      x.out_stride = q;
      x.k = gq.m[a].e.kc;
      x.v = gq.m[a].e.vc;
      al[a] = lv;
    }
    TP_TRY(attn_tree_group(aa, al, na, st));
    TP_TRY(sk_gemm_group(go, po, st));
    ::tp::count_launch(), rmsnorm_group_kernel<<<dim3(maxn, na), kNormThreads, 0, st>>>(ng, d, c.norm_eps);
    TP_CUDA(cudaGetLastError());
    TP_TRY(sk_gemm_group(ggu, pgu, st));
    TP_TRY(sk_gemm_group(gdn, pdn, st));
    // input norm of the next slot, for the members that continue
    int nc = 0;
    NormGroup nn;
    int maxc = 0;
    for (int a = 0; a < na; ++a)
      if (lvs[idx[a]].layer_lo + j + 1 < lvs[idx[a]].layer_hi) {
        nn.x[nc] = ng.x[a];
        nn.xd[nc] = ng.xd[a];
        nn.n[nc] = ng.n[a];
        maxc = std::max(maxc, ng.n[a]);
        ++nc;
      }
    if (nc) {
      ::tp::count_launch(), rmsnorm_group_kernel<<<dim3(maxc, nc), kNormThreads, 0, st>>>(nn, d, c.norm_eps);
      TP_CUDA(cudaGetLastError());
    }
  }
  return TP_OK;
}

}  // namespace tp
