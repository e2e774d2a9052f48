// Llama-shape stage compute: bf16 weights in HBM, fp32 residual stream.
//
// Per layer (reference layer_step structure, `/root/reference/pkg/src/treepipe/
// model.py:250-280`, with the Llama block: RMSNorm, RoPE, GQA, SwiGLU), with the
// RMSNorms folded into the GEMMs (no norm kernels):
//
//   QKV  = r . (Xd . Wqkv^T)   K2 (epilogue: scale by the node's r, RoPE(q,k); q -> Xq;
//                                 k,v -> paged KV rows in place)
//   attn = tree-attention(Xq, KV, ancestor bits)      K1 (attn.cu, 2 launches) -> Xo
//   x   += Xo . Wo^T           K2 (epilogue: residual add; Xd = bf16(x); per (node,
//                                 m-tile) sums of squares -> r of the next GEMM)
//   Xf   = silu(r G) * (r U)   K2 over the gate/up weights (64-row interleave)
//   x   += Xf . Wdown^T        K2 (epilogue: residual add, Xd = bf16(x) and the sums
//                                 of squares for the next layer's QKV)
//
// 6 launches per layer (plus one prep launch per forward call, which writes the
// first layer's Xd and sums of squares); every kernel is a programmatic-dependent
// launch whose prologue overlaps the preceding kernel where resources allow.
//
// Numerics (mirrored by oracle/llama.py): GEMM inputs bf16, accumulation and
// residual fp32; r = 1/sqrt(mean(x^2) + eps) applied to the fp32 GEMM output;
// RoPE (HF rotate-half, angle in fp64) on the fp32 output, then rounded to bf16
// for the cache / attention; softmax fp32.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>

#include "attn.h"
#include "gemm_tc.h"
#include "internal.h"

namespace tp {

enum { kCtrQkv = 0, kCtrO, kCtrGu, kCtrDown, kCtrHead, kCtrKinds };

// Transient scratch of one member of a (grouped) forward: node-row operands of
// the GEMMs, stream-K partials / counters, RoPE table, attention partials.
// Owned by the model (a small pool, one per member slot of a grouped launch),
// not by the stages, so hundreds of request caches carry no scratch.
struct LlamaWs {
  int np = 0;  // padded node rows (multiple of 16)
  __nv_bfloat16 *Xd = nullptr, *Xo = nullptr, *Xf = nullptr, *Xq = nullptr;
  __nv_bfloat16 *kself = nullptr, *vself = nullptr;
  float* part = nullptr;
  size_t part_floats = 0;
  int* counters = nullptr;  // [kCtrKinds][ctr_stride]
  int ctr_stride = 0;
  float* rope = nullptr;  // [np][64][2]
  float* ssp = nullptr;   // [np][d / 128] RMSNorm partials of the rows in Xd (folded norm)
  CUtensorMap mXd, mXo, mXf;
  CUtensorMap mXq3;  // query rows for the attention run kernel (make_tmap_q3d)
  float *pm = nullptr, *pl = nullptr, *po = nullptr;
  int max_chunks = 0;
};

struct LlamaModelExt {
  std::vector<CUtensorMap> qkv, o, gu, down;
  CUtensorMap head;
  std::vector<LlamaWs*> ws;  // member workspaces
  std::mutex mu;             // host-side enqueue of one forward at a time (worker threads)
  std::map<std::pair<const void*, int>, cudaGraphExec_t> graphs;  // (stage, layer slots) -> the layer loop's graph
  int32_t* d_tok = nullptr;  // greedy tokens of a multi-row verify
  int32_t* h_tok = nullptr;  // pinned
  cudaEvent_t tok_ev = nullptr;
};

static LlamaModelExt* mext(tp_model* m) { return reinterpret_cast<LlamaModelExt*>(m->tma_cache); }

// ---- kernels --------------------------------------------------------------------

__global__ void llama_embed_kernel(const __nv_bfloat16* __restrict__ E, const int32_t* __restrict__ tok, int d,
                                   float* __restrict__ x) {
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
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

// Batched per-item helpers of a forward call (one launch each instead of one per item).
constexpr int kMaxBatchItems = 64;
struct RowCopyGroup {
  const float* src[kMaxBatchItems];
  float* dst[kMaxBatchItems];
  __nv_bfloat16* xd[kMaxBatchItems];  // the first layer's RMSNorm output (nullptr: none)
  int rows[kMaxBatchItems];
  int d[kMaxBatchItems];  // the item's model width
  float* ssp[kMaxBatchItems];  // the first layer's RMSNorm partials [rows][d / 128] (with xd)
};
// token rows of several items -> their residual-stream rows (fp32), one launch
struct EmbedGroup {
  const int32_t* tok[kMaxBatchItems];
  float* out[kMaxBatchItems];
  __nv_bfloat16* xd[kMaxBatchItems];  // the first layer's RMSNorm output (nullptr: none)
  int n[kMaxBatchItems];
  const __nv_bfloat16* E[kMaxBatchItems];  // the item's model's embedding table
  int d[kMaxBatchItems];
  float* ssp[kMaxBatchItems];
};
// hidden rows handed over from the previous stage -> the member's residual stream

struct RopeGroup {
  const int32_t* pos[kMaxBatchItems];
  float* out[kMaxBatchItems];
  int n[kMaxBatchItems];
  double theta[kMaxBatchItems];
};

// The prep of a forward call as ONE launch (each a separate grid before: every
// launch in the PDL chain costs a grid-completion hop): blockIdx.y selects an
// embedding item, a hidden-row copy item or a RoPE-table item; the per-task
// arithmetic of each task is unchanged (bf16 -> fp32 row, float4 row copy, f64 RoPE angles).
struct PrepGroup {
  EmbedGroup e;
  RowCopyGroup c;
  RopeGroup r;
  int ne, nc, nr;
};
__global__ void __launch_bounds__(1024) prep_group_kernel(const __grid_constant__ PrepGroup P) {
  pdl_wait();
  pdl_trigger();
  int y = blockIdx.y;
  const int x = blockIdx.x;
  if (y < P.ne + P.nc) {  // one residual-stream row (+ its first layer's bf16 operand and RMSNorm partials)
    const bool emb = y < P.ne;
    const int k = emb ? y : y - P.ne;
    if (x >= (emb ? P.e.n[k] : P.c.rows[k])) return;
    const int d = emb ? P.e.d[k] : P.c.d[k];
    float* o = (emb ? P.e.out[k] : P.c.dst[k]) + (size_t)x * d;
    __nv_bfloat16* xd = emb ? P.e.xd[k] : P.c.xd[k];
    float v[kNormPer];
    if (emb) {
      const __nv_bfloat16* e = P.e.E[k] + (size_t)P.e.tok[k][x] * d;
#pragma unroll
      for (int u = 0; u < kNormPer; ++u) {
        const int j = threadIdx.x + u * 1024;
        v[u] = j < d ? __bfloat162float(e[j]) : 0.f;
      }
    } else {
      const float* src = P.c.src[k] + (size_t)x * d;
#pragma unroll
      for (int u = 0; u < kNormPer; ++u) {
        const int j = threadIdx.x + u * 1024;
        v[u] = j < d ? src[j] : 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < kNormPer; ++u) {
      const int j = threadIdx.x + u * 1024;
      if (j < d) o[j] = v[u];
    }
    if (xd) {  // bf16(x) and the per-128-column sums of squares, exactly as the residual epilogue
      float* ssp = emb ? P.e.ssp[k] : P.c.ssp[k];
      __syncthreads();  // the row's fp32 values are in global memory
      const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
      for (int mt = w; mt * 128 < d; mt += 32) {
        const float4 vv = *reinterpret_cast<const float4*>(o + mt * 128 + 4 * l);
        st_bf16x4(xd + (size_t)x * d + mt * 128 + 4 * l, vv.x, vv.y, vv.z, vv.w);
        const float s = tile_sumsq(vv);
        if (l == 0) ssp[(size_t)x * (d / 128) + mt] = s;
      }
    }
    return;
  }
  y -= P.ne + P.nc;
  const int i = threadIdx.x;
  if (x >= P.r.n[y] || i >= 64) return;
  const double inv = pow(P.r.theta[y], -2.0 * (double)i / 128.0);
  double sn, cs;
  sincos((double)P.r.pos[y][x] * inv, &sn, &cs);
  P.r.out[y][((size_t)x * 64 + i) * 2] = (float)cs;
  P.r.out[y][((size_t)x * 64 + i) * 2 + 1] = (float)sn;
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

static void ws_free(LlamaWs* e) {
  if (!e) return;
  for (void* p : {(void*)e->Xd, (void*)e->Xo, (void*)e->Xf, (void*)e->Xq, (void*)e->kself, (void*)e->vself,
                  (void*)e->part, (void*)e->counters, (void*)e->rope, (void*)e->ssp, (void*)e->pm, (void*)e->pl,
                  (void*)e->po})
    if (p) cudaFree(p);
  delete e;
}

void llama_model_free(tp_model* m) {
  LlamaModelExt* me = mext(m);
  if (!me) return;
  for (LlamaWs* e : me->ws) ws_free(e);
  for (auto& kv : me->graphs)
    if (kv.second) cudaGraphExecDestroy(kv.second);
  if (me->d_tok) cudaFree(me->d_tok);
  if (me->h_tok) cudaFreeHost(me->h_tok);
  if (me->tok_ev) cudaEventDestroy(me->tok_ev);
  delete me;
  m->tma_cache = nullptr;
}

int llama_workspace_bytes(const tp_model*, int, size_t* bytes) {
  *bytes = 256;  // llama scratch lives in the model workspace pool (llama.cu)
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

// Workspace g of the model's pool, grown to hold `min_chunks` attention chunks.
static int ws_get(tp_model* m, int g, int min_chunks, LlamaWs** out) {
  LlamaModelExt* me = mext(m);
  const tp_model_config& c = m->cfg;
  while ((int)me->ws.size() <= g) me->ws.push_back(nullptr);
  LlamaWs*& e = me->ws[g];
  if (e == nullptr) {
    e = new LlamaWs();
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
    TP_CUDA(cudaMalloc(&e->ssp, np * (d / 128) * 4));
    TP_CUDA(cudaMemset(e->ssp, 0, np * (d / 128) * 4));
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
    sk_counters_forget(e->counters, (size_t)kCtrKinds * e->ctr_stride * 4);
    TP_TRY(make_tmap_kmajor(&e->mXd, e->Xd, np, d, 16));
    TP_TRY(make_tmap_q3d(&e->mXq3, e->Xq, np, c.heads, c.heads / c.kv_heads));
    TP_TRY(make_tmap_kmajor(&e->mXo, e->Xo, np, q, 16));
    TP_TRY(make_tmap_kmajor(&e->mXf, e->Xf, np, f, 16));
  }
  if (min_chunks > e->max_chunks) {
    // grows with the largest KV capacity seen (rare): drain in-flight users first
    TP_CUDA(cudaDeviceSynchronize());
    if (e->pm) cudaFree(e->pm);
    if (e->pl) cudaFree(e->pl);
    if (e->po) cudaFree(e->po);
    const int chunks = std::max(min_chunks, 2 * e->max_chunks);
    const size_t cells = (size_t)e->np * c.heads * chunks;
    TP_CUDA(cudaMalloc(&e->pm, cells * 4));
    TP_CUDA(cudaMalloc(&e->pl, cells * 4));
    TP_CUDA(cudaMalloc(&e->po, cells * 128 * 4));
    e->max_chunks = chunks;
  }
  *out = e;
  return TP_OK;
}

static int chunks_for_cap(int cap) { return (cap + kAttnMaxExtra + 1 + kAttnChunk - 1) / kAttnChunk; }

int llama_stage_init(tp_stage* s) { return build_model_ext(s->m); }

void llama_stage_free(tp_stage*) {}

int llama_embed(tp_model* m, int n, const int32_t* d_tokens, float* out, cudaStream_t st) {
  TP_CHECK(m->embed, TP_ECONFIG, "model has no embedding table");
  ::tp::count_launch();
  TP_CUDA(launch_pdl(llama_embed_kernel, dim3(n), dim3(256), 0, st, (const __nv_bfloat16*)m->embed, d_tokens,
                     (int)m->cfg.hidden, out));
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

static GemmEpi epi_base(LlamaWs* e, int kind) {
  GemmEpi g;
  g.part = e->part;
  g.counters = e->counters + (size_t)kind * e->ctr_stride;
  return g;
}

static int logits_locked(tp_model* m, int n, const float* x, float* logits, cudaStream_t st) {
  TP_CHECK(m->head, TP_ECONFIG, "model has no LM head");
  TP_TRY(build_model_ext(m));
  LlamaWs* e;
  TP_TRY(ws_get(m, 0, 1, &e));
  const int d = m->cfg.hidden, V = m->cfg.vocab;
  ::tp::count_launch();
  TP_CUDA(launch_pdl(rmsnorm_kernel, dim3(n), dim3(kNormThreads), 0, st, x, d, m->cfg.norm_eps, e->Xd));
  TP_CUDA(cudaGetLastError());
  GemmEpi g = epi_base(e, kCtrHead);
  g.op = kOpStore;
  g.out = logits;
  g.out_ld = V;
  return sk_gemm(&mext(m)->head, &e->mXd, sk_plan(V, d, n), g, st);
}

int llama_logits(tp_model* m, tp_stage*, int n, const float* x, float* logits, cudaStream_t st) {
  TP_TRY(build_model_ext(m));
  std::lock_guard<std::mutex> lk(mext(m)->mu);
  return logits_locked(m, n, x, logits, st);
}

int llama_greedy_rows_async(tp_model* m, int n, const float* x, float* logits, cudaStream_t st) {
  TP_TRY(build_model_ext(m));
  LlamaModelExt* me = mext(m);
  std::lock_guard<std::mutex> lk(me->mu);
  if (!me->d_tok) {
    TP_CUDA(cudaMalloc(&me->d_tok, 4 * (size_t)std::max(64, m->cfg.max_nodes)));
    TP_CUDA(cudaMallocHost(&me->h_tok, 4 * (size_t)std::max(64, m->cfg.max_nodes)));
    TP_CUDA(cudaEventCreateWithFlags(&me->tok_ev, cudaEventDisableTiming));
  }
  TP_TRY(logits_locked(m, n, x, logits, st));
  TP_TRY(argmax_rows(logits, m->cfg.vocab, n, me->d_tok, st));
  timeline_mark("verify_head", st);
  TP_CUDA(cudaMemcpyAsync(me->h_tok, me->d_tok, 4 * (size_t)n, cudaMemcpyDeviceToHost, st));
  TP_CUDA(cudaEventRecord(me->tok_ev, st));
  return TP_OK;
}

int llama_greedy_rows_wait(tp_model* m, int n, int32_t* out) {
  LlamaModelExt* me = mext(m);
  TP_CHECK(me && me->tok_ev, TP_ECONFIG, "no multi-row verify in flight");
  TP_CUDA(cudaEventSynchronize(me->tok_ev));
  std::memcpy(out, me->h_tok, 4 * (size_t)n);
  return TP_OK;
}

int llama_forward(tp_stage* s, const LevelDev& lv, const void* hidden_in, void* hidden_out, cudaStream_t st) {
  FwdItem it{s, lv, hidden_in};
  FwdMember mb{&it, 1, (float*)hidden_out};
  return llama_forward_members(&mb, 1, st, 0);
}

// Members of a grouped forward run layer slot by layer slot: slot j runs layer
// lo_g + j of every member g that has one, each GEMM as ONE grouped launch over
// the members (same segment boundaries as ungrouped launches, so every member's
// bits equal its stand-alone forward).  A member is a ragged batch of items —
// one request each (SpecPipe-DB) — that share the member's layers: their node
// rows are concatenated for the GEMMs (weights streamed once for all requests),
// K/V rows are scattered to each request's cache, and attention runs per item.
// Diagnostics only (tp_debug_attn_knob 3): skip kernel classes in the layer loop
// to measure each one's marginal cost inside the PDL chain — results are WRONG
// while set.  Bits: 1 attention, 4 GEMMs (2, the RMSNorm kernels, no longer exists: folded).
int g_dbg_skip = 0;
// Diagnostics only (tp_debug_dump): device buffer receiving member 0's slot-0
// intermediates of the next forward call: Xd (input RMSNorm, bf16 n x d), Xq
// (RoPE'd queries, bf16 n x q), Xo (attention out, bf16 n x q), x after
// the o-projection (f32 n x d), Xd (post-attention RMSNorm, bf16 n x d),
// Xf (SwiGLU product, bf16 n x f), x after the down projection (f32 n x d).
void* g_dbg_dump = nullptr;

// TP_GRAPH=1 turns the graph mode on.  Measured on a shard stream, a lone 4-layer 7B
// stage: 153 -> 88 us of host time per forward call, 406 -> 398 us of GPU time; but
// the emulated 8-GPU bench (8 shards on one GPU) shows no end-to-end change (same
// box: 5.34 / 5.41 vs 5.35 / 5.33 ms/token), so it stays opt-in.
bool g_graph_env = getenv("TP_GRAPH") && atoi(getenv("TP_GRAPH")) != 0;  // also tp_debug_attn_knob(5, on)
std::atomic<long long> g_graph_launches{0};  // graph replays (tp_graph_launches)
bool timeline_on();
bool gemm_profile_on();

static bool graph_mode_ok(int count, const FwdMember* mem, cudaStream_t st) {
  // the legacy default stream cannot be captured (stage-per-GPU shard streams can)
  return g_graph_env && st != nullptr && st != cudaStreamLegacy && st != cudaStreamPerThread && count == 1 &&
         mem[0].count == 1 && !g_dbg_skip && !g_dbg_dump && !timeline_on() && !gemm_profile_on();
}

int llama_forward_members(const FwdMember* mem, int count, cudaStream_t st, int ws_base) {
  TP_CHECK(count >= 1 && count <= kMaxGroup, TP_ECONFIG, "member group size outside [1, 8]");
  // Members may belong to different model objects of the same device (a draft
  // model's level grouped with a target stage's): every shape, weight and
  // workspace below is the member's own model's; each model's enqueue lock is
  // taken once, in address order.
  tp_model* mg[kMaxGroup];
  std::vector<tp_model*> models;
  for (int g = 0; g < count; ++g) {
    mg[g] = mem[g].items[0].s->m;
    TP_TRY(build_model_ext(mg[g]));
    if (std::find(models.begin(), models.end(), mg[g]) == models.end()) models.push_back(mg[g]);
  }
  std::sort(models.begin(), models.end());
  std::vector<std::unique_lock<std::mutex>> locks;
  for (tp_model* m : models) locks.emplace_back(mext(m)->mu);
  LlamaWs* ws[kMaxGroup];
  std::vector<int> offs[kMaxGroup];
  struct Copy {
    const float* src;
    float* dst;
    __nv_bfloat16* xd;
    int rows, d;
    float* ssp;
  };
  std::vector<Copy> copies;
  struct Embed {
    const int32_t* tok;
    float* out;
    __nv_bfloat16* xd;
    int n;
    const __nv_bfloat16* E;
    int d;
    float* ssp;
  };
  std::vector<Embed> embeds;
  int ntot[kMaxGroup], lo[kMaxGroup], hi[kMaxGroup];
  int slots = 0;
  for (int g = 0; g < count; ++g) {
    const FwdMember& M = mem[g];
    const tp_model_config& c = mg[g]->cfg;
    const int d = c.hidden;
    TP_CHECK(M.count >= 1 && M.x, TP_ECONFIG, "empty forward member");
    int cap_max = 1, n = 0;
    lo[g] = M.items[0].lv.layer_lo;
    hi[g] = M.items[0].lv.layer_hi;
    for (int r = 0; r < M.count; ++r) {
      const FwdItem& it = M.items[r];
      TP_CHECK(it.s->m == mg[g], TP_ECONFIG, "the items of a member must share one model object");
      TP_CHECK(it.lv.layer_lo == lo[g] && it.lv.layer_hi == hi[g], TP_ECONFIG,
               "items of a member must run the same layers");
      cap_max = std::max(cap_max, it.s->cap);
      offs[g].push_back(n);
      n += it.lv.n;
    }
    TP_CHECK(n <= c.max_nodes, TP_ESHAPE, "ragged member exceeds max_nodes");
    ntot[g] = n;
    TP_TRY(ws_get(mg[g], ws_base + g, chunks_for_cap(cap_max), &ws[g]));
    for (int r = 0; r < M.count; ++r) {
      const FwdItem& it = M.items[r];
      float* x = M.x + (size_t)offs[g][r] * d;
      // the first layer's GEMM operand bf16(x) and RMSNorm partials come from the prep
      // launch (rows in place are "copied" onto themselves so that every row gets them)
      __nv_bfloat16* xd = hi[g] > lo[g] ? ws[g]->Xd + (size_t)offs[g][r] * d : nullptr;
      float* ssp = ws[g]->ssp + (size_t)offs[g][r] * (d / 128);
      if (it.hin) {
        if (it.hin != x || xd) copies.push_back({(const float*)it.hin, x, xd, it.lv.n, d, ssp});
      } else {
        TP_CHECK(mg[g]->embed, TP_ECONFIG, "model has no embedding table");
        embeds.push_back({it.lv.tokens, x, xd, it.lv.n, (const __nv_bfloat16*)mg[g]->embed, d, ssp});
      }
    }
    slots = std::max(slots, hi[g] - lo[g]);
  }
  {  // embeddings, hidden-row copies and RoPE tables of every item: one launch per 64 of each kind
    struct Rope {
      const int32_t* pos;
      float* out;
      int n;
      double theta;
    };
    std::vector<Rope> ropes;
    for (int g = 0; g < count && slots > 0; ++g) {
      if (hi[g] == lo[g]) continue;
      for (int r = 0; r < mem[g].count; ++r) {
        const FwdItem& it = mem[g].items[r];
        ropes.push_back({it.lv.positions, ws[g]->rope + (size_t)offs[g][r] * 128, it.lv.n,
                         (double)mg[g]->cfg.rope_theta});
      }
    }
    size_t ie = 0, ic = 0, ir = 0;
    while (ie < embeds.size() || ic < copies.size() || ir < ropes.size()) {
      PrepGroup P;
      P.ne = (int)std::min<size_t>(kMaxBatchItems, embeds.size() - ie);
      P.nc = (int)std::min<size_t>(kMaxBatchItems, copies.size() - ic);
      P.nr = (int)std::min<size_t>(kMaxBatchItems, ropes.size() - ir);
      int mx = 1;
      for (int k = 0; k < P.ne; ++k) {
        const Embed& e = embeds[ie + k];
        P.e.tok[k] = e.tok;
        P.e.out[k] = e.out;
        P.e.xd[k] = e.xd;
        P.e.n[k] = e.n;
        P.e.E[k] = e.E;
        P.e.d[k] = e.d;
        P.e.ssp[k] = e.ssp;
        mx = std::max(mx, e.n);
      }
      for (int k = 0; k < P.nc; ++k) {
        const Copy& cp = copies[ic + k];
        P.c.src[k] = cp.src;
        P.c.dst[k] = cp.dst;
        P.c.xd[k] = cp.xd;
        P.c.rows[k] = cp.rows;
        P.c.d[k] = cp.d;
        P.c.ssp[k] = cp.ssp;
        mx = std::max(mx, cp.rows);
      }
      for (int k = 0; k < P.nr; ++k) {
        P.r.pos[k] = ropes[ir + k].pos;
        P.r.out[k] = ropes[ir + k].out;
        P.r.n[k] = ropes[ir + k].n;
        P.r.theta[k] = ropes[ir + k].theta;
        mx = std::max(mx, P.r.n[k]);
      }
      ::tp::count_launch();
      TP_CUDA(launch_pdl(prep_group_kernel, dim3(mx, P.ne + P.nc + P.nr), dim3(1024), 0, st, P));
      ie += P.ne;
      ic += P.nc;
      ir += P.nr;
    }
  }
  if (slots == 0) return TP_OK;
  // per-request KV destinations of ragged members (one small upload each)
  const QkvItem* qitems[kMaxGroup] = {nullptr};
  const int32_t* qnode[kMaxGroup] = {nullptr};
  for (int g = 0; g < count; ++g) {
    const FwdMember& M = mem[g];
    if (hi[g] == lo[g]) continue;
    if (M.count > 1) {
      std::vector<char> blob(sizeof(QkvItem) * M.count + 4 * (size_t)ntot[g]);
      QkvItem* qi = reinterpret_cast<QkvItem*>(blob.data());
      int32_t* ni = reinterpret_cast<int32_t*>(blob.data() + sizeof(QkvItem) * M.count);
      for (int r = 0; r < M.count; ++r) {
        const FwdItem& it = M.items[r];
        qi[r] = QkvItem{it.s->d_ptab, it.s->max_pages, it.s->lo, it.lv.row0, it.lv.append, offs[g][r]};
        for (int i = 0; i < it.lv.n; ++i) ni[offs[g][r] + i] = r;
      }
      const char* dptr;
      TP_TRY(upload(M.items[0].s, blob.data(), blob.size(), st, &dptr));
      qitems[g] = reinterpret_cast<const QkvItem*>(dptr);
      qnode[g] = reinterpret_cast<const int32_t*>(dptr + sizeof(QkvItem) * M.count);
    }
  }
  // each member's plans (one set per distinct shape; identical to its ungrouped launches)
  SkPlan pqkv[kMaxGroup], po[kMaxGroup], pgu[kMaxGroup], pdn[kMaxGroup];
  for (int g = 0; g < count; ++g) {
    const tp_model_config& c = mg[g]->cfg;
    const int q = c.heads * 128, kvd = c.kv_heads * 128;
    pqkv[g] = sk_plan(q + 2 * kvd, c.hidden, 1);
    po[g] = sk_plan(c.hidden, q, 1);
    pgu[g] = sk_plan(2 * c.ffn, c.hidden, 1);
    pdn[g] = sk_plan(c.hidden, c.ffn, 1);
  }
  timeline_mark("fwd_prep", st);
  auto run_slots = [&]() -> int {
  std::vector<AttnArgs> aa;
  std::vector<LevelDev> al;
  for (int j = 0; j < slots; ++j) {
    int idx[kMaxGroup], na = 0;
    for (int g = 0; g < count; ++g)
      if (lo[g] + j < hi[g]) idx[na++] = g;
    GemmGroup gq, go, ggu, gdn;
    gq.count = go.count = ggu.count = gdn.count = na;
    int mx = 16;
    aa.clear();
    al.clear();
    for (int a = 0; a < na; ++a) {
      const int g = idx[a];
      const FwdMember& M = mem[g];
      const tp_model_config& c = mg[g]->cfg;
      LlamaModelExt* me = mext(mg[g]);
      const int d = c.hidden, H = c.heads, KV = c.kv_heads, f = c.ffn;
      const int q = H * 128, kvd = KV * 128;
      LlamaWs* e = ws[g];
      const int layer = lo[g] + j, li = layer - c.layer_lo;
      const int n = ntot[g], npad = std::max(16, (n + 15) / 16 * 16);
      mx = std::max(mx, npad);
      const FwdItem& i0 = M.items[0];
      // RMSNorm folded into the GEMMs: the residual epilogues (o, down) write bf16(x)
      // and per-m-tile sums of squares; qkv and gate/up scale their rows by r
      auto norm_in = [&](GemmEpi& ep) {
        ep.ssp_in = e->ssp;
        ep.ssp_ld = ep.ssp_n = d / 128;
        ep.norm_d = (float)d;
        ep.norm_eps = c.norm_eps;
      };
      GemmEpi eq = epi_base(e, kCtrQkv);
      norm_in(eq);
      eq.op = kOpQkv;
      eq.H = H;
      eq.KV = KV;
      eq.rope = e->rope;
      eq.xq = e->Xq;
      eq.kself = e->kself;
      eq.vself = e->vself;
      eq.layer = layer;
      if (M.count == 1) {
        eq.row0 = i0.lv.row0;
        eq.append = i0.lv.append;
        eq.ptab = i0.s->d_ptab + (size_t)(layer - i0.s->lo) * i0.s->max_pages;
      } else {
        eq.items = qitems[g];
        eq.node_item = qnode[g];
      }
      GemmEpi er = epi_base(e, kCtrO);
      er.op = kOpResid;
      er.out = M.x;
      er.out_ld = d;
      er.xd_out = e->Xd;
      er.xd_ld = d;
      er.ssp_out = e->ssp;
      er.ssp_ld = d / 128;
      GemmEpi ed = er;
      ed.counters = e->counters + (size_t)kCtrDown * e->ctr_stride;
      if (layer + 1 >= hi[g]) ed.xd_out = nullptr, ed.ssp_out = nullptr;  // the stage's last layer: no consumer
      GemmEpi eg = epi_base(e, kCtrGu);
      norm_in(eg);
      eg.op = kOpSwiglu;
      eg.xf = e->Xf;
      eg.f = f;
      auto set = [&](GemmGroup& gg, const CUtensorMap& wa, const CUtensorMap& xb, const GemmEpi& ep,
                     const SkPlan& p) {
        gg.m[a].a = wa;
        gg.m[a].b = xb;
        gg.m[a].e = ep;
        gg.m[a].n = n;
        gg.m[a].n_pad = npad;
        gg.m[a].p = p;
      };
      set(gq, me->qkv[li], e->mXd, eq, pqkv[g]);
      set(go, me->o[li], e->mXo, er, po[g]);
      set(ggu, me->gu[li], e->mXd, eg, pgu[g]);
      set(gdn, me->down[li], e->mXf, ed, pdn[g]);
      for (int r = 0; r < M.count; ++r) {
        const FwdItem& it = M.items[r];
        const size_t off = offs[g][r];
        AttnArgs x;
        x.q = e->Xq + off * q;
        x.q_stride = q;
        x.qmap = e->mXq3;
        x.q_row0 = (int)off;
        x.ptab = it.s->d_ptab + (size_t)(layer - it.s->lo) * it.s->max_pages;
        x.cap = it.s->cap;
        x.kself = it.lv.append ? nullptr : e->kself + off * kvd;
        x.vself = it.lv.append ? nullptr : e->vself + off * kvd;
        x.H = H;
        x.KV = KV;
        x.scale = (float)(1.0 / std::sqrt(128.0));
        x.pm = e->pm + off * H * e->max_chunks;
        x.pl = e->pl + off * H * e->max_chunks;
        x.po = e->po + off * H * e->max_chunks * 128;
        x.max_chunks = e->max_chunks;
        x.out = e->Xo + off * q;
        x.out_stride = q;
        aa.push_back(x);
        al.push_back(it.lv);
      }
    }
    gq.max_npad = go.max_npad = ggu.max_npad = gdn.max_npad = mx;
    // (slot 0's input RMSNorm ran inside the prep launch)
    char* dump = (j == 0 && g_dbg_dump) ? static_cast<char*>(g_dbg_dump) : nullptr;
    const int g0 = idx[0];
    const size_t dn = (size_t)ntot[g0];
    const size_t dd = mg[g0]->cfg.hidden, dq = (size_t)mg[g0]->cfg.heads * 128, df = mg[g0]->cfg.ffn;
    auto dump_cp = [&](const void* src, size_t bytes) -> int {
      if (!dump) return TP_OK;
      TP_CUDA(cudaMemcpyAsync(dump, src, bytes, cudaMemcpyDeviceToDevice, st));
      dump += bytes;
      return TP_OK;
    };
    TP_TRY(dump_cp(ws[g0]->Xd, dn * dd * 2));
    if (!(g_dbg_skip & 4)) TP_TRY(sk_gemm_group(gq, st));
    timeline_mark("gemm_qkv", st);
    TP_TRY(dump_cp(ws[g0]->Xq, dn * dq * 2));
    for (size_t a0 = 0; a0 < aa.size() && !(g_dbg_skip & 1); a0 += kAttnMaxGroup) {
      const int cnt = (int)std::min<size_t>(kAttnMaxGroup, aa.size() - a0);
      TP_TRY(attn_tree_group(aa.data() + a0, al.data() + a0, cnt, st));
    }
    TP_TRY(dump_cp(ws[g0]->Xo, dn * dq * 2));
    if (!(g_dbg_skip & 4)) TP_TRY(sk_gemm_group(go, st));
    timeline_mark("gemm_o", st);
    TP_TRY(dump_cp(mem[g0].x, dn * dd * 4));
    TP_TRY(dump_cp(ws[g0]->Xd, dn * dd * 2));
    if (!(g_dbg_skip & 4)) TP_TRY(sk_gemm_group(ggu, st));
    timeline_mark("gemm_gate_up", st);
    TP_TRY(dump_cp(ws[g0]->Xf, dn * df * 2));
    if (!(g_dbg_skip & 4)) TP_TRY(sk_gemm_group(gdn, st));
    timeline_mark("gemm_down", st);
    TP_TRY(dump_cp(mem[g0].x, dn * dd * 4));
    if (dump) g_dbg_dump = nullptr;
  }
  return TP_OK;
  };
  // CUDA-graph mode (TP_GRAPH=1; a lone single-request member on a capturable
  // stream, i.e. the stage-per-GPU shard streams): the layer loop's
  // launches are captured and replayed through one graph launch, the executable
  // graph updated in place from each call's fresh capture (same topology: the
  // kernels' arguments — node counts, cache rows, K2 epochs — change per call).
  if (graph_mode_ok(count, mem, st)) {
    std::vector<int*> ctr;
    for (int g = 0; g < count; ++g)
      for (int k = 0; k < kCtrKinds; ++k) ctr.push_back(ws[g]->counters + (size_t)k * ws[g]->ctr_stride);
    std::vector<int> saved = sk_epochs_get(ctr);
    TP_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    const int rc = run_slots();
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(st, &graph);
    if (rc != TP_OK || ce != cudaSuccess || !graph) {  // nothing ran: roll the epochs back, launch directly
      static bool told = false;
      if (!told && getenv("TP_GRAPH_DEBUG")) {
        fprintf(stderr, "[tp graph] capture failed: rc=%d end=%s (%s)\n", rc, cudaGetErrorString(ce),
                tp_last_error());
        told = true;
      }
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      sk_epochs_set(ctr, saved);
      return run_slots();
    }
    cudaGraphExec_t& exec = mext(mg[0])->graphs[std::make_pair((const void*)mem[0].items[0].s, slots)];
    bool ok = false;
    if (exec) {
      cudaGraphExecUpdateResultInfo info;
      ok = cudaGraphExecUpdate(exec, graph, &info) == cudaSuccess;
      if (!ok) {
        cudaGetLastError();
        cudaGraphExecDestroy(exec);
        exec = nullptr;
      }
    }
    if (!ok && cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) exec = nullptr;
    cudaGraphDestroy(graph);
    if (exec) g_graph_launches.fetch_add(1, std::memory_order_relaxed);
    if (!exec || cudaGraphLaunch(exec, st) != cudaSuccess) {  // the capture never ran: same fallback
      cudaGetLastError();
      if (exec) cudaGraphExecDestroy(exec);
      exec = nullptr;
      sk_epochs_set(ctr, saved);
      return run_slots();
    }
    return TP_OK;
  }
  return run_slots();
}

}  // namespace tp

extern "C" int tp_graph_launches(int64_t* n) {
  *n = tp::g_graph_launches.load();
  return TP_OK;
}
