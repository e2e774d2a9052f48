// C-ABI of libtreepipe_b200.so (see include/treepipe_b200.h for the contract and
// the reference call each entry point replaces).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>

#include "attn.h"
#include "gemm_tc.h"
#include "internal.h"

#include <atomic>
#include <cstdlib>

namespace tp {
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
static std::atomic<long long> g_launches{0};
static std::atomic<long long> g_h2d{0}, g_d2h{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
static void count_io(long long h2d, long long d2h) {
  g_h2d.fetch_add(h2d, std::memory_order_relaxed);
  g_d2h.fetch_add(d2h, std::memory_order_relaxed);
}
}  // namespace tp

// ---- optional GPU timeline: events between kernel groups, aggregated per tag ----
namespace tp {
struct TlRec {
  const char* tag;
  cudaEvent_t ev;
  cudaStream_t st;
};
static std::vector<TlRec> g_tl;
static bool g_tl_on = false;
static std::mutex g_tl_mu;
bool timeline_on() { return g_tl_on; }

void timeline_mark(const char* tag, cudaStream_t st) {
  if (!g_tl_on) return;
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return;
  cudaEventRecord(e, st);
  std::lock_guard<std::mutex> g(g_tl_mu);
  g_tl.push_back({tag, e, st});
}
}  // namespace tp

namespace tp {
extern int g_dbg_skip;
extern bool g_graph_env;
extern void* g_dbg_dump;
}

extern "C" int tp_debug_attn_tile(int32_t on) {
  // the experimental 16-node tile path was removed (measured slower); only "off" remains valid
  return on ? TP_ECONFIG : TP_OK;
}

extern "C" int tp_debug_dump(void* dev_buf) {
  tp::g_dbg_dump = dev_buf;
  return TP_OK;
}

extern "C" int tp_debug_attn_trace(void* dev_buf) { return tp::attn_set_trace(dev_buf); }

extern "C" int tp_debug_attn_knob(int32_t knob, int32_t value) {
  if (knob == 3) {
    tp::g_dbg_skip = value;
    return TP_OK;
  }
  if (knob == 1) return tp::attn_set_run(value);
  if (knob == 5) {  // CUDA-graph mode of lone forwards on capturable streams (llama.cu)
    tp::g_graph_env = value != 0;
    return TP_OK;
  }
  // knobs 0 (tile path) and 2 (shared-prefix tail) were removed
  return (knob == 0 || knob == 2) && value == 0 ? TP_OK : TP_ECONFIG;
}

// K4 on caller logits (tests): n_rows == 1 with children -> argmax + first matching
// child (argmax_match_kernel); otherwise the per-row first argmax (fp32 only).
extern "C" int tp_debug_argmax(int32_t device, const void* logits_dev, int32_t is_f64, int32_t vocab, int32_t n_rows,
                               const int32_t* children_host, int32_t n_children, int32_t* out_host) {
  TP_CUDA(cudaSetDevice(device));
  TP_CHECK(logits_dev && out_host && vocab >= 1 && n_rows >= 1, TP_ECONFIG, "bad argmax arguments");
  int32_t* d = nullptr;
  const size_t words = (size_t)std::max(n_rows, 2) + (size_t)std::max(n_children, 0);
  TP_CUDA(cudaMalloc(&d, words * 4));
  int rc = TP_OK;
  if (children_host && n_rows == 1) {
    int32_t* dch = d + 2;
    if (n_children > 0) TP_CUDA(cudaMemcpy(dch, children_host, (size_t)n_children * 4, cudaMemcpyHostToDevice));
    rc = tp::argmax_match(logits_dev, is_f64, vocab, dch, n_children, d, 0);
    if (rc == TP_OK) TP_CUDA(cudaMemcpy(out_host, d, 8, cudaMemcpyDeviceToHost));
  } else {
    TP_CHECK(!is_f64, TP_ECONFIG, "per-row argmax is fp32");
    rc = tp::argmax_rows(logits_dev, vocab, n_rows, d, 0);
    if (rc == TP_OK) TP_CUDA(cudaMemcpy(out_host, d, (size_t)n_rows * 4, cudaMemcpyDeviceToHost));
  }
  cudaFree(d);
  return rc;
}

extern "C" int tp_timeline_enable(int32_t on) {
  tp::g_tl_on = on != 0;
  return TP_OK;
}

// "tag=ms;tag=ms;..." : GPU time from the previous mark on the same stream to
// each mark, summed per tag; resets the record.
extern "C" int tp_timeline_read(char* buf, int32_t len) {
  std::lock_guard<std::mutex> g(tp::g_tl_mu);
  std::vector<std::pair<std::string, double>> acc;
  for (size_t i = 0; i < tp::g_tl.size(); ++i) {
    auto& r = tp::g_tl[i];
    cudaEventSynchronize(r.ev);
    for (size_t j = i; j-- > 0;)
      if (tp::g_tl[j].st == r.st) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, tp::g_tl[j].ev, r.ev);
        bool found = false;
        for (auto& a : acc)
          if (a.first == r.tag) {
            a.second += ms;
            found = true;
          }
        if (!found) acc.push_back({r.tag, ms});
        break;
      }
  }
  for (auto& r : tp::g_tl) cudaEventDestroy(r.ev);
  tp::g_tl.clear();
  std::string out;
  for (auto& a : acc) out += a.first + "=" + std::to_string(a.second) + ";";
  std::snprintf(buf, (size_t)len, "%s", out.c_str());
  return TP_OK;
}

extern "C" int tp_launch_count(int64_t* out) {
  *out = tp::g_launches.load();
  return TP_OK;
}

extern "C" int tp_io_bytes(int64_t* h2d, int64_t* d2h) {
  *h2d = tp::g_h2d.load();
  *d2h = tp::g_d2h.load();
  return TP_OK;
}

using namespace tp;

namespace tp {
// Claim the next staging slot (waiting only if the stream has not yet executed
// the upload that last used it); returns host + device addresses of the slot.
int meta_slot(tp_stage* s, size_t bytes, char** host, char** dev, int* slot) {
  TP_CHECK(bytes <= s->meta_bytes, TP_ESHAPE, "metadata exceeds stage staging buffer");
  const int k = s->meta_next;
  s->meta_next = (k + 1) % tp_stage::kMetaRing;
  TP_CUDA(cudaEventSynchronize(s->meta_ev[k]));
  *host = s->host_meta + (size_t)k * s->meta_bytes;
  *dev = s->meta + (size_t)k * s->meta_bytes;
  *slot = k;
  return TP_OK;
}

int meta_push(tp_stage* s, int slot, size_t bytes, cudaStream_t st) {
  const size_t off = (size_t)slot * s->meta_bytes;
  TP_CUDA(cudaMemcpyAsync(s->meta + off, s->host_meta + off, bytes, cudaMemcpyHostToDevice, st));
  count_io((long long)bytes, 0);
  TP_CUDA(cudaEventRecord(s->meta_ev[slot], st));
  return TP_OK;
}

int upload(tp_stage* s, const void* host, size_t bytes, cudaStream_t st, const char** dev_out) {
  char *h, *d;
  int k;
  TP_TRY(meta_slot(s, bytes, &h, &d, &k));
  std::memcpy(h, host, bytes);
  TP_TRY(meta_push(s, k, bytes, st));
  *dev_out = d;
  return TP_OK;
}

}  // namespace tp

namespace {

struct ToyTensorSpec {
  int64_t rows, cols;
};

// toy per-layer tensors in generation order (model.py:224-233)
ToyTensorSpec toy_spec(int d, int which) {
  switch (which) {
    case 1: case 2: case 3: case 4: return {d, d};
    case 5: return {d, 2 * d};
    case 6: return {2 * d, d};
  }
  return {0, 0};
}

size_t meta_capacity(const tp_model* m, int cap, int* words) {
  *words = (cap + 64) / 64 + 1;
  size_t n = (size_t)std::max(m->cfg.max_nodes, 64);
  size_t bytes = n * 4 * 4                       // tokens, positions, prefix rows, children
                 + n * (size_t)(*words) * 8      // anc bits
                 + n * (size_t)(65 * 4) + 16     // decoded ancestor rows [n][<=64] + counts
                 + (size_t)(cap + 64) * 4        // compaction / gather index lists
                 + 256;
  return (bytes + 255) & ~(size_t)255;
}

// Llama pages from the model's pool (kvpage.cuh): slabs of >= 64 MB, zeroed once
// (stale rows of recycled pages are finite; the attention kernel multiplies the
// rows past a chunk's end by exact zeros).
int page_take(tp_model* m, size_t count, char** out) {
  std::lock_guard<std::mutex> lk(m->pool_mu);
  if (m->page_free.size() < count) {
    const int64_t pb = page_bytes(m->cfg.kv_heads);
    const size_t want = std::max<size_t>(count - m->page_free.size(), (size_t)std::max<int64_t>(1, (64LL << 20) / pb));
    void* slab = nullptr;
    TP_CUDA(cudaMalloc(&slab, want * pb));
    TP_CUDA(cudaMemset(slab, 0, want * pb));
    m->page_slabs.push_back(slab);
    for (size_t i = 0; i < want; ++i) m->page_free.push_back(static_cast<char*>(slab) + i * pb);
  }
  for (size_t i = 0; i < count; ++i) {
    out[i] = m->page_free.back();
    m->page_free.pop_back();
  }
  return TP_OK;
}

// Grow a Llama stage to >= cap rows by appending pages to every hosted layer.
int alloc_pages(tp_stage* s, int cap) {
  const int nl = s->hi - s->lo;
  const int have = s->cap / kPageRows, need = (cap + kPageRows - 1) / kPageRows;
  if (need > have && nl > 0) {
    if (need > s->max_pages) {  // the table itself grows (rare): in-flight kernels may read the old one
      const int mp = std::max(need, std::max(16, 2 * s->max_pages));
      std::vector<char*> t((size_t)nl * mp, nullptr);
      for (int l = 0; l < nl; ++l)
        for (int p = 0; p < have; ++p) t[(size_t)l * mp + p] = s->ptab[(size_t)l * s->max_pages + p];
      s->ptab.swap(t);
      if (s->d_ptab) {
        TP_CUDA(cudaDeviceSynchronize());
        cudaFree(s->d_ptab);
      }
      TP_CUDA(cudaMalloc((void**)&s->d_ptab, sizeof(char*) * (size_t)nl * mp));
      s->max_pages = mp;
    }
    std::vector<char*> fresh((size_t)nl * (need - have));
    TP_TRY(page_take(s->m, fresh.size(), fresh.data()));
    size_t k = 0;
    for (int l = 0; l < nl; ++l)
      for (int p = have; p < need; ++p) s->ptab[(size_t)l * s->max_pages + p] = fresh[k++];
    // entries below `have` are unchanged, so kernels still reading them are unaffected
    TP_CUDA(cudaMemcpy(s->d_ptab, s->ptab.data(), sizeof(char*) * s->ptab.size(), cudaMemcpyHostToDevice));
  }
  s->cap = std::max(have, need) * kPageRows;
  return TP_OK;
}

int alloc_kv(tp_stage* s, int cap) {
  int nl = s->hi - s->lo;
  if (s->m->cfg.arch != TP_ARCH_TOY) {
    TP_TRY(alloc_pages(s, cap));
    cap = s->cap;
  } else {
    size_t plane = (size_t)s->kv_heads * cap * s->head_dim * s->esize;
    std::vector<void*> k(nl), v(nl);
    for (int l = 0; l < nl; ++l) {
      TP_CUDA(cudaMalloc(&k[l], plane));
      TP_CUDA(cudaMalloc(&v[l], plane));
      TP_CUDA(cudaMemset(k[l], 0, plane));
      TP_CUDA(cudaMemset(v[l], 0, plane));
      if (!s->k.empty()) {  // reserve(): carry rows over, head plane by head plane
        size_t row = (size_t)s->head_dim * s->esize;
        for (int h = 0; h < s->kv_heads; ++h) {
          TP_CUDA(cudaMemcpy((char*)k[l] + h * cap * row, (char*)s->k[l] + h * (size_t)s->cap * row,
                             (size_t)s->rows * row, cudaMemcpyDeviceToDevice));
          TP_CUDA(cudaMemcpy((char*)v[l] + h * cap * row, (char*)s->v[l] + h * (size_t)s->cap * row,
                             (size_t)s->rows * row, cudaMemcpyDeviceToDevice));
        }
        cudaFree(s->k[l]);
        cudaFree(s->v[l]);
      }
    }
    s->k = k;
    s->v = v;
    s->cap = cap;
    std::vector<void*> planes(2 * nl);
    for (int l = 0; l < nl; ++l) {
      planes[2 * l] = k[l];
      planes[2 * l + 1] = v[l];
    }
    if (s->d_planes) cudaFree(s->d_planes);
    TP_CUDA(cudaMalloc(&s->d_planes, sizeof(void*) * std::max(1, 2 * nl)));
    if (nl) TP_CUDA(cudaMemcpy(s->d_planes, planes.data(), sizeof(void*) * 2 * nl, cudaMemcpyHostToDevice));
  }
  // metadata staging follows capacity
  if (s->meta) cudaFree(s->meta);
  if (s->host_meta) cudaFreeHost(s->host_meta);
  s->meta_bytes = meta_capacity(s->m, cap, &s->max_words);
  TP_CUDA(cudaMalloc((void**)&s->meta, s->meta_bytes * tp_stage::kMetaRing));
  TP_CUDA(cudaMallocHost((void**)&s->host_meta, s->meta_bytes * tp_stage::kMetaRing));
  return TP_OK;
}

bool is_toy(const tp_model* m) { return m->cfg.arch == TP_ARCH_TOY; }

}  // namespace

namespace tp {
KvView kv_view(const tp_stage* s) {
  KvView v{};
  v.heads = s->kv_heads;
  v.row_bytes = s->head_dim * s->esize;
  if (is_toy(s->m)) {
    v.tab = reinterpret_cast<char* const*>(s->d_planes);
    v.paged = 0;
    v.plane_stride = (int64_t)s->cap * v.row_bytes;
  } else {
    v.tab = s->d_ptab;
    v.paged = 1;
    v.max_pages = s->max_pages;
  }
  return v;
}
}  // namespace tp

extern "C" {

const char* tp_last_error(void) { return g_err.c_str(); }

int tp_device_count(int32_t* out) {
  int n = 0;
  TP_CUDA(cudaGetDeviceCount(&n));
  *out = n;
  return TP_OK;
}

int tp_model_create(const tp_model_config* cfg, tp_model** out) {
  TP_CHECK(cfg && out, TP_ECONFIG, "null argument");
  const tp_model_config& c = *cfg;
  TP_CHECK(c.arch == TP_ARCH_TOY || c.arch == TP_ARCH_LLAMA, TP_ECONFIG, "unknown arch");
  TP_CHECK(c.vocab >= 16, TP_ESHAPE, "vocab must be at least 16");
  TP_CHECK(c.hidden >= 2 && c.hidden % 2 == 0, TP_ESHAPE, "hidden dim must be even");
  TP_CHECK(c.layers >= 1, TP_ESHAPE, "need at least one layer");
  TP_CHECK(0 <= c.layer_lo && c.layer_lo <= c.layer_hi && c.layer_hi <= c.layers, TP_ECONFIG,
           "hosted layer range outside the model");
  TP_CHECK(c.max_nodes >= 1 && c.max_nodes <= 1024, TP_ECONFIG, "max_nodes must lie in [1, 1024]");
  // a Llama forward is one K2 GEMM per layer slot over all of a member's rows
  TP_CHECK(c.arch != TP_ARCH_LLAMA || c.max_nodes <= 256, TP_ECONFIG,
           "Llama max_nodes must lie in [1, 256] (rows per K2 GEMM)");
  TP_CUDA(cudaSetDevice(c.device));
  tp_model* m = new tp_model();
  m->cfg = c;
  int rc = TP_OK;
  const int64_t d = c.hidden, V = c.vocab;
  if (is_toy(m)) {
    m->cfg.heads = m->cfg.kv_heads = 1;
    m->cfg.head_dim = c.hidden;
    m->cfg.ffn = 2 * c.hidden;
    if (c.with_embed || c.with_head) {
      m->embed_bytes = V * d * 8;
      if (cudaMalloc(&m->embed, m->embed_bytes) != cudaSuccess) rc = TP_ECUDA;
    }
    for (int l = c.layer_lo; l < c.layer_hi && rc == TP_OK; ++l) {
      tp_layer_weights w;
      for (int t = 1; t <= 6; ++t) {
        ToyTensorSpec sp = toy_spec((int)d, t);
        w.bytes[t] = sp.rows * sp.cols * 8;
        if (cudaMalloc(&w.w[t], w.bytes[t]) != cudaSuccess) rc = TP_ECUDA;
      }
      m->layers.push_back(w);
    }
  } else {
    TP_CHECK(c.heads >= 1 && c.kv_heads >= 1 && c.heads % c.kv_heads == 0, TP_ESHAPE,
             "heads must be a multiple of kv_heads");
    TP_CHECK(c.head_dim == 128, TP_ESHAPE, "llama path supports head_dim 128");
    TP_CHECK(c.hidden % 128 == 0 && c.ffn % 128 == 0, TP_ESHAPE, "hidden and ffn must be multiples of 128");
    const int64_t q = (int64_t)c.heads * c.head_dim, kv = (int64_t)c.kv_heads * c.head_dim, f = c.ffn;
    if (c.with_embed) {
      m->embed_bytes = V * d * 2;
      if (cudaMalloc(&m->embed, m->embed_bytes) != cudaSuccess) rc = TP_ECUDA;
    }
    if (c.with_head) {
      m->head_bytes = V * d * 2;
      if (cudaMalloc(&m->head, m->head_bytes) != cudaSuccess) rc = TP_ECUDA;
    }
    for (int l = c.layer_lo; l < c.layer_hi && rc == TP_OK; ++l) {
      tp_layer_weights w;
      w.bytes[1] = (q + 2 * kv) * d * 2;  // fused [Wq; Wk; Wv]  ([out, in])
      w.bytes[4] = d * q * 2;             // Wo
      w.bytes[5] = 2 * f * d * 2;         // fused gate/up, 64-row interleave
      w.bytes[7] = d * f * 2;             // Wdown
      for (int t : {1, 4, 5, 7})
        if (cudaMalloc(&w.w[t], w.bytes[t]) != cudaSuccess) rc = TP_ECUDA;
      m->layers.push_back(w);
    }
  }
  if (rc != TP_OK) {
    set_error("cudaMalloc failed while allocating weights");
    tp_model_destroy(m);
    return rc;
  }
  *out = m;
  return TP_OK;
}

static void stage_release(tp_stage* s);
static void model_free_now(tp_model* m);

int tp_model_destroy(tp_model* m) {
  if (!m) return TP_OK;
  std::vector<tp_stage*> parked;
  bool now;
  {
    std::lock_guard<std::mutex> lk(m->pool_mu);
    parked.swap(m->stage_pool);
    now = m->live_stages == 0;
    m->destroy_pending = !now;
  }
  cudaSetDevice(m->cfg.device);
  for (tp_stage* s : parked) stage_release(s);
  if (now) model_free_now(m);
  return TP_OK;
}

static void model_free_now(tp_model* m) {
  cudaSetDevice(m->cfg.device);
  if (m->embed) cudaFree(m->embed);
  if (m->head) cudaFree(m->head);
  for (auto& w : m->layers)
    for (void* p : w.w)
      if (p) cudaFree(p);
  if (!is_toy(m)) llama_model_free(m);
  call_ring_free(m);
  if (m->prune_plan) cudaFree(m->prune_plan);
  for (void* p : m->page_slabs) cudaFree(p);
  delete m;
}

int tp_model_init_lcg(tp_model* m, uint64_t seed, void* stream) {
  TP_CUDA(cudaSetDevice(m->cfg.device));
  cudaStream_t st = (cudaStream_t)stream;
  if (!is_toy(m)) {
    TP_TRY(llama_init_weights(m, seed, st));
    TP_CUDA(cudaStreamSynchronize(st));
    return TP_OK;
  }
  const int64_t d = m->cfg.hidden, V = m->cfg.vocab;
  const int64_t per_layer = 8 * d * d;
  if (m->embed) TP_TRY(lcg_fill_f64((double*)m->embed, V * d, seed, 0, st));
  for (int l = m->cfg.layer_lo; l < m->cfg.layer_hi; ++l) {
    int64_t off = V * d + (int64_t)l * per_layer;
    const tp_layer_weights& w = m->layers[l - m->cfg.layer_lo];
    for (int t = 1; t <= 6; ++t) {
      int64_t cnt = w.bytes[t] / 8;
      TP_TRY(lcg_fill_f64((double*)w.w[t], cnt, seed, off, st));
      off += cnt;
    }
  }
  TP_CUDA(cudaStreamSynchronize(st));
  return TP_OK;
}

int tp_lcg_uniform(int32_t device, uint64_t seed, int64_t start, int64_t count, void* out_dev, void* stream) {
  TP_CUDA(cudaSetDevice(device));
  TP_CHECK(count >= 0 && start >= 0, TP_ESHAPE, "negative range");
  if (count == 0) return TP_OK;
  return lcg_fill_f64((double*)out_dev, count, seed, start, (cudaStream_t)stream);
}

static int tensor_ptr(const tp_model* m, int which, int layer, void** p, int64_t* bytes) {
  if (which == 0) {
    *p = m->embed;
    *bytes = m->embed_bytes;
  } else if (which == 8 && !is_toy(m)) {
    *p = m->head;
    *bytes = m->head_bytes;
  } else {
    TP_CHECK(layer >= m->cfg.layer_lo && layer < m->cfg.layer_hi, TP_ESHAPE, "layer not hosted by model");
    TP_CHECK(which >= 1 && which <= 7, TP_ESHAPE, "bad tensor id");
    const tp_layer_weights& w = m->layers[layer - m->cfg.layer_lo];
    *p = w.w[which];
    *bytes = w.bytes[which];
  }
  TP_CHECK(*p != nullptr, TP_ESHAPE, "tensor not present (llama tensors are fused: ids 1,4,5,7)");
  return TP_OK;
}

int tp_model_tensor_bytes(const tp_model* m, int32_t which, int32_t layer, int64_t* nbytes) {
  void* p;
  return tensor_ptr(m, which, layer, &p, nbytes);
}

int tp_model_write_tensor(tp_model* m, int32_t which, int32_t layer, const void* host, int64_t nbytes) {
  TP_CUDA(cudaSetDevice(m->cfg.device));
  void* p;
  int64_t b;
  TP_TRY(tensor_ptr(m, which, layer, &p, &b));
  TP_CHECK(b == nbytes, TP_ESHAPE, "tensor size mismatch");
  TP_CUDA(cudaMemcpy(p, host, b, cudaMemcpyHostToDevice));
  return TP_OK;
}

int tp_model_read_tensor(const tp_model* m, int32_t which, int32_t layer, void* host, int64_t nbytes) {
  TP_CUDA(cudaSetDevice(m->cfg.device));
  void* p;
  int64_t b;
  TP_TRY(tensor_ptr(m, which, layer, &p, &b));
  TP_CHECK(b == nbytes, TP_ESHAPE, "tensor size mismatch");
  TP_CUDA(cudaMemcpy(host, p, b, cudaMemcpyDeviceToHost));
  return TP_OK;
}

static void stage_release(tp_stage* s);
static constexpr size_t kStagePoolMax = 64;

int tp_stage_create(tp_model* m, int32_t layer_lo, int32_t layer_hi, int32_t capacity_rows, tp_stage** out) {
  TP_CHECK(m && out, TP_ECONFIG, "null argument");
  TP_CHECK(m->cfg.layer_lo <= layer_lo && layer_lo <= layer_hi && layer_hi <= m->cfg.layer_hi, TP_ECONFIG,
           "stage layers must be hosted by the model");
  TP_CHECK(capacity_rows >= 1, TP_ECONFIG, "capacity must be positive");
  TP_CUDA(cudaSetDevice(m->cfg.device));
  {  // reuse a parked stage of the same shape (no allocation, no device sync)
    std::lock_guard<std::mutex> lk(m->pool_mu);
    for (size_t i = 0; i < m->stage_pool.size(); ++i) {
      tp_stage* p = m->stage_pool[i];
      if (p->lo == layer_lo && p->hi == layer_hi && p->cap >= capacity_rows && p->cap <= 4 * capacity_rows) {
        m->stage_pool.erase(m->stage_pool.begin() + (long)i);
        p->rows = 0;
        ++m->live_stages;
        *out = p;
        return TP_OK;
      }
    }
  }
  tp_stage* s = new tp_stage();
  s->m = m;
  s->lo = layer_lo;
  s->hi = layer_hi;
  if (is_toy(m)) {
    s->kv_heads = 1;
    s->head_dim = m->cfg.hidden;
    s->esize = 8;
    TP_TRY(toy_workspace_bytes(m, m->cfg.max_nodes, &s->ws_bytes));
  } else {
    s->kv_heads = m->cfg.kv_heads;
    s->head_dim = m->cfg.head_dim;
    s->esize = 2;
    TP_TRY(llama_workspace_bytes(m, m->cfg.max_nodes, &s->ws_bytes));
  }
  int rc = alloc_kv(s, capacity_rows);
  if (rc != TP_OK) {
    stage_release(s);  // partially built: free, never park
    return rc;
  }
  TP_CUDA(cudaMalloc((void**)&s->ws, s->ws_bytes));
  TP_CUDA(cudaMemset(s->ws, 0, s->ws_bytes));
  for (auto& ev : s->meta_ev) {
    TP_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    TP_CUDA(cudaEventRecord(ev, 0));
  }
  TP_CUDA(cudaEventCreateWithFlags(&s->verify_ev, cudaEventDisableTiming));
  TP_CUDA(cudaMalloc((void**)&s->d_result, 16));
  TP_CUDA(cudaMallocHost((void**)&s->h_result, 16));
  TP_CUDA(cudaMalloc(&s->logits, (size_t)m->cfg.vocab * 8));
  s->logits_rows = 1;
  if (!is_toy(m)) {
    rc = llama_stage_init(s);
    if (rc != TP_OK) {
      stage_release(s);
      return rc;
    }
  }
  {
    std::lock_guard<std::mutex> lk(m->pool_mu);
    ++m->live_stages;
  }
  *out = s;
  return TP_OK;
}

static void stage_release(tp_stage* s);

int tp_stage_destroy(tp_stage* s) {
  if (!s) return TP_OK;
  tp_model* m = s->m;
  bool release, free_model = false;
  tp_stage* evict = nullptr;
  {
    std::lock_guard<std::mutex> lk(m->pool_mu);
    --m->live_stages;
    release = m->destroy_pending;
    if (!release) {
      m->stage_pool.push_back(s);  // parked: reused, or freed with the model
      // bounded: past kStagePoolMax parked stages the oldest is really freed
      // (one device sync, instead of memory growing with every finished request)
      if (m->stage_pool.size() > kStagePoolMax) {
        evict = m->stage_pool.front();
        m->stage_pool.erase(m->stage_pool.begin());
      }
    }
    free_model = release && m->live_stages == 0;
  }
  if (evict) stage_release(evict);
  if (release) stage_release(s);
  if (free_model) model_free_now(m);
  return TP_OK;
}

static void stage_release(tp_stage* s) {
  cudaSetDevice(s->m->cfg.device);
  for (void* p : s->k) cudaFree(p);
  for (void* p : s->v) cudaFree(p);
  {  // pages go back to the model's pool
    std::lock_guard<std::mutex> lk(s->m->pool_mu);
    for (char* p : s->ptab)
      if (p) s->m->page_free.push_back(p);
  }
  if (s->d_ptab) cudaFree(s->d_ptab);
  if (s->ws) cudaFree(s->ws);
  if (s->meta) cudaFree(s->meta);
  if (s->host_meta) cudaFreeHost(s->host_meta);
  for (auto ev : s->meta_ev)
    if (ev) cudaEventDestroy(ev);
  if (s->verify_ev) cudaEventDestroy(s->verify_ev);
  if (s->d_result) cudaFree(s->d_result);
  if (s->h_result) cudaFreeHost(s->h_result);
  if (s->d_planes) cudaFree(s->d_planes);
  if (s->logits) cudaFree(s->logits);
  if (!is_toy(s->m)) llama_stage_free(s);
  delete s;
}

int tp_stage_rows(const tp_stage* s, int32_t* rows) {
  *rows = s->rows;
  return TP_OK;
}

int tp_stage_reserve(tp_stage* s, int32_t capacity_rows) {
  if (capacity_rows <= s->cap) return TP_OK;
  TP_CUDA(cudaSetDevice(s->m->cfg.device));
  TP_CUDA(cudaDeviceSynchronize());  // the metadata ring follows the capacity (re-allocated)
  TP_TRY(alloc_kv(s, capacity_rows));
  return is_toy(s->m) ? TP_OK : llama_stage_init(s);
}

}  // extern "C"

// Validate one level against its stage, upload its metadata (one pinned-host ->
// device copy) and describe it for the kernels.
// Tree-form levels: derive prefix_rows / anc_bits from the tree's packed rows
// (self bit cleared, promoted ancestors below tree_off masked) into `store`.
struct LevelStore {
  std::vector<int32_t> pre;
  std::vector<uint64_t> bits;
};
static const tp_level* materialize(const tp_level* L, tp_level* tmp, LevelStore* store) {
  if (!L->tree_bits) return L;
  *tmp = *L;
  const int n = L->n, W = L->words;
  store->pre.assign(n, L->tree_prefix);
  store->bits.assign((size_t)n * W, 0ull);
  for (int i = 0; i < n; ++i) {
    const int node = L->tree_lo + i;
    const uint64_t* src = L->tree_bits + (size_t)node * W;
    uint64_t* dst = store->bits.data() + (size_t)i * W;
    for (int w = 0; w < W; ++w) {
      uint64_t v = src[w];
      if (w == (node >> 6)) v &= ~(1ull << (node & 63));  // self
      const int lo_bit = L->tree_off - 64 * w;            // tree nodes below tree_off live in the prefix
      if (lo_bit >= 64) v = 0;
      else if (lo_bit > 0) v &= ~((1ull << lo_bit) - 1ull);
      dst[w] = v;
    }
  }
  tmp->prefix_rows = store->pre.data();
  tmp->anc_bits = W ? store->bits.data() : nullptr;
  tmp->bits_base = L->tree_prefix - L->tree_off;
  tmp->tree_bits = nullptr;
  return tmp;
}

// Validate one level against its stage and describe it for the kernels; the
// metadata blob (tokens | positions | prefix | anc bits | anc counts | anc rows)
// is laid out by level_write into caller-provided staging memory.
static int level_validate(tp_stage* s, const tp_level* L, const void* hidden_in, void* hidden_out, LevelDev* out,
                          size_t* bytes) {
  TP_CHECK(s && L && hidden_out, TP_ECONFIG, "null argument");
  tp_model* m = s->m;
  const int n = L->n;
  TP_CHECK(n >= 1 && n <= m->cfg.max_nodes, TP_ESHAPE, "level size outside [1, max_nodes]");
  TP_CHECK(L->positions && L->prefix_rows, TP_ECONFIG, "positions and prefix_rows are required");
  TP_CHECK(hidden_in || (L->tokens && m->embed), TP_ECONFIG, "need hidden_in or tokens + embedding");
  TP_CHECK(L->words >= 0 && L->words <= s->max_words, TP_ESHAPE, "too many mask words for this stage");
  TP_CHECK(!L->append || s->rows + n <= s->cap, TP_ESHAPE, "KV capacity exceeded (reserve first)");
  const int visible = s->rows + (L->append ? n : 0);
  int max_t = 0, uniform_a = -2, a_max = 0;
  for (int i = 0; i < n; ++i) {
    int pc = 0;
    for (int w = 0; w < L->words; ++w) pc += __builtin_popcountll(L->anc_bits[(int64_t)i * L->words + w]);
    if (uniform_a == -2) uniform_a = pc;
    else if (uniform_a != pc || L->prefix_rows[i] != L->prefix_rows[0]) uniform_a = -1;
    // Llama attention: the node-specific ancestors live in the last 16-slot window (attn.cu)
    TP_CHECK(is_toy(m) || pc <= 15, TP_ESHAPE, "more than 15 speculative ancestors per node");
    (void)a_max;
    max_t = std::max(max_t, L->prefix_rows[i] + pc + 1);
    TP_CHECK(L->prefix_rows[i] >= 0 && L->prefix_rows[i] <= visible, TP_ECONTRACT, "prefix rows beyond cache");
    if (L->tokens && !hidden_in)
      TP_CHECK(L->tokens[i] >= 0 && L->tokens[i] < m->cfg.vocab, TP_ESHAPE, "token outside vocabulary");
    for (int w = 0; w < L->words; ++w) {
      uint64_t bits = L->anc_bits[(int64_t)i * L->words + w];
      if (!bits) continue;
      int hi_bit = 63 - __builtin_clzll(bits), lo_bit = __builtin_ctzll(bits);
      TP_CHECK(L->bits_base + w * 64 + lo_bit >= 0 && L->bits_base + w * 64 + hi_bit < visible, TP_ECONTRACT,
               "ancestor row outside the cache");
    }
  }
  LevelDev lv{};
  lv.n = n;
  lv.append = L->append;
  lv.row0 = s->rows;
  lv.words = L->words;
  lv.bits_base = L->bits_base;
  lv.max_t = max_t;
  lv.min_p = *std::min_element(L->prefix_rows, L->prefix_rows + n);
  lv.uniform_a = uniform_a;
  lv.anc_stride = a_max;
  const bool all_layers = L->layer_lo == 0 && L->layer_hi == 0;
  const bool no_layers = L->layer_lo < 0;  // explicit empty range: embed/copy only
  lv.layer_lo = all_layers ? s->lo : (no_layers ? s->lo : L->layer_lo);
  lv.layer_hi = all_layers ? s->hi : (no_layers ? s->lo : L->layer_hi);
  TP_CHECK(s->lo <= lv.layer_lo && lv.layer_lo <= lv.layer_hi && lv.layer_hi <= s->hi, TP_ESHAPE,
           "layer range not hosted by this stage");
  const size_t off_anc = ((12 * (size_t)n) + 7) & ~(size_t)7;
  *bytes = (off_anc + 8 * (size_t)n * L->words + 4 * (size_t)n + 4 * (size_t)n * a_max + 15) & ~(size_t)15;
  *out = lv;
  return TP_OK;
}

static void level_write(const tp_level* L, LevelDev* lv, char* h, const char* dm) {
  const int n = L->n, a_max = lv->anc_stride;
  const size_t off_tok = 0, off_pos = 4 * (size_t)n, off_pre = 8 * (size_t)n;
  const size_t off_anc = ((12 * (size_t)n) + 7) & ~(size_t)7;
  const size_t off_cnt = off_anc + 8 * (size_t)n * L->words;
  const size_t off_rows = off_cnt + 4 * (size_t)n;
  if (L->tokens) std::memcpy(h + off_tok, L->tokens, 4 * (size_t)n);
  else std::memset(h + off_tok, 0, 4 * (size_t)n);
  std::memcpy(h + off_pos, L->positions, 4 * (size_t)n);
  std::memcpy(h + off_pre, L->prefix_rows, 4 * (size_t)n);
  if (L->words) std::memcpy(h + off_anc, L->anc_bits, 8 * (size_t)n * L->words);
  // per-node ancestor counts; the rows themselves are decoded from the bit-rows on
  // the device (attn.cu ancestor_row)
  int32_t* cnt = reinterpret_cast<int32_t*>(h + off_cnt);
  for (int i = 0; i < n; ++i) {
    int k = 0;
    for (int w = 0; w < L->words; ++w) k += __builtin_popcountll(L->anc_bits[(int64_t)i * L->words + w]);
    cnt[i] = k;
  }
  lv->tokens = (const int32_t*)(dm + off_tok);
  lv->positions = (const int32_t*)(dm + off_pos);
  lv->prefix_rows = (const int32_t*)(dm + off_pre);
  lv->anc = (const uint64_t*)(dm + off_anc);
  lv->anc_cnt = (const int32_t*)(dm + off_cnt);
  lv->anc_rows = (const int32_t*)(dm + off_rows);
}

// One level through its stage's own staging ring.
static int prepare_level(tp_stage* s, const tp_level* L, const void* hidden_in, void* hidden_out, cudaStream_t st,
                         LevelDev* out) {
  size_t bytes;
  TP_TRY(level_validate(s, L, hidden_in, hidden_out, out, &bytes));
  char *h, *dm;
  int slot;
  TP_TRY(meta_slot(s, bytes, &h, &dm, &slot));
  level_write(L, out, h, dm);
  return meta_push(s, slot, bytes, st);
}

// Per-model staging ring for calls that carry several levels / index lists at
// once: one pinned-host -> device copy per call instead of one per stage.
namespace tp {
struct CallRing {
  static constexpr int kSlots = 8;
  char* host = nullptr;
  char* dev = nullptr;
  size_t slot_bytes = 0;
  cudaEvent_t ev[kSlots] = {nullptr};    // copy of the slot complete (host buffer reusable)
  cudaEvent_t free_[kSlots] = {nullptr}; // compute stream past the slot's readers (device buffer reusable)
  cudaStream_t copy = nullptr;           // side copy stream (default; TP_SIDE_COPY=0 copies on the compute stream)
  cudaStream_t last_st = nullptr;        // the compute stream of the previous call
  int next = 0, last = -1;
  bool side = false;
};

int call_slot(tp_model* m, size_t bytes, char** host, char** dev, int* slot) {
  auto* r = reinterpret_cast<CallRing*>(m->call_ring);
  if (!r) {
    r = new CallRing();
    m->call_ring = r;
    for (auto& e : r->ev) {
      TP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      TP_CUDA(cudaEventRecord(e, 0));
    }
    for (auto& e : r->free_) {
      TP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      TP_CUDA(cudaEventRecord(e, 0));
    }
    r->side = !(getenv("TP_SIDE_COPY") && atoi(getenv("TP_SIDE_COPY")) == 0);
    if (r->side) TP_CUDA(cudaStreamCreateWithFlags(&r->copy, cudaStreamNonBlocking));
  }
  if (bytes > r->slot_bytes) {  // grow (rare): drain users of the old buffers first
    TP_CUDA(cudaDeviceSynchronize());
    if (r->host) cudaFreeHost(r->host);
    if (r->dev) cudaFree(r->dev);
    r->slot_bytes = std::max<size_t>(bytes, (size_t)1 << 20);
    TP_CUDA(cudaMallocHost((void**)&r->host, r->slot_bytes * CallRing::kSlots));
    TP_CUDA(cudaMalloc((void**)&r->dev, r->slot_bytes * CallRing::kSlots));
  }
  const int k = r->next;
  r->next = (k + 1) % CallRing::kSlots;
  TP_CUDA(cudaEventSynchronize(r->ev[k]));
  *host = r->host + (size_t)k * r->slot_bytes;
  *dev = r->dev + (size_t)k * r->slot_bytes;
  *slot = k;
  return TP_OK;
}

int call_push(tp_model* m, int slot, size_t bytes, cudaStream_t st) {
  auto* r = reinterpret_cast<CallRing*>(m->call_ring);
  const size_t off = (size_t)slot * r->slot_bytes;
  if (r->side) {
    // Metadata copies run on a side copy stream: the compute stream only waits for
    // this slot's copy (typically long done) instead of serialising a memcpy node
    // behind all of its previous kernels.  The previous call's readers are all
    // enqueued on its compute stream by now: mark that slot reusable there.
    if (r->last >= 0) TP_CUDA(cudaEventRecord(r->free_[r->last], r->last_st));
    r->last = slot;
    r->last_st = st;
    if (bytes) {
      TP_CUDA(cudaStreamWaitEvent(r->copy, r->free_[slot], 0));  // this slot's earlier readers are done
      TP_CUDA(cudaMemcpyAsync(r->dev + off, r->host + off, bytes, cudaMemcpyHostToDevice, r->copy));
      count_io((long long)bytes, 0);
    }
    TP_CUDA(cudaEventRecord(r->ev[slot], r->copy));
    TP_CUDA(cudaStreamWaitEvent(st, r->ev[slot], 0));
    return TP_OK;
  }
  if (bytes) {
    TP_CUDA(cudaMemcpyAsync(r->dev + off, r->host + off, bytes, cudaMemcpyHostToDevice, st));
    count_io((long long)bytes, 0);
  }
  TP_CUDA(cudaEventRecord(r->ev[slot], st));
  return TP_OK;
}

void call_ring_free(tp_model* m) {
  auto* r = reinterpret_cast<CallRing*>(m->call_ring);
  if (!r) return;
  if (r->host) cudaFreeHost(r->host);
  if (r->dev) cudaFree(r->dev);
  for (auto e : r->ev)
    if (e) cudaEventDestroy(e);
  for (auto e : r->free_)
    if (e) cudaEventDestroy(e);
  if (r->copy) cudaStreamDestroy(r->copy);
  delete r;
  m->call_ring = nullptr;
}
}  // namespace tp

extern "C" {

int tp_stage_forward(tp_stage* s, const tp_level* L, const void* hidden_in, void* hidden_out, void* stream) {
  TP_CHECK(s && L && hidden_out, TP_ECONFIG, "null argument");
  tp_model* m = s->m;
  TP_CUDA(cudaSetDevice(m->cfg.device));
  cudaStream_t st = (cudaStream_t)stream;
  tp_level tmp;
  LevelStore store;
  L = materialize(L, &tmp, &store);
  LevelDev lv;
  TP_TRY(prepare_level(s, L, hidden_in, hidden_out, st, &lv));
  int rc = is_toy(m) ? toy_forward(s, lv, hidden_in, hidden_out, st) : llama_forward(s, lv, hidden_in, hidden_out, st);
  if (rc != TP_OK) return rc;
  if (L->append) s->rows += L->n;
  return TP_OK;
}

int tp_stages_forward(int32_t count, tp_stage* const* stages, const tp_level* levels, const void* const* hidden_in,
                      void* const* hidden_out, void* stream) {
  TP_CHECK(count >= 1 && stages && levels && hidden_in && hidden_out, TP_ECONFIG, "null argument");
  std::vector<tp_item> items(count);
  for (int g = 0; g < count; ++g) items[g] = tp_item{stages[g], levels[g], hidden_in[g], g};
  return tp_items_forward(count, items.data(), hidden_out, stream);
}

int tp_items_forward(int32_t n_items, const tp_item* items, void* const* member_hidden_out, void* stream) {
  return tp_items_forward_ws(n_items, items, member_hidden_out, 0, stream);
}

int tp_items_forward_ws(int32_t n_items, const tp_item* items, void* const* member_hidden_out, int32_t ws_base,
                        void* stream) {
  TP_CHECK(ws_base >= 0 && ws_base <= 64, TP_ECONFIG, "workspace base outside [0, 64]");
  TP_CHECK(n_items >= 1 && items && member_hidden_out, TP_ECONFIG, "null argument");
  tp_model* m0 = items[0].stage ? items[0].stage->m : nullptr;
  TP_CHECK(m0, TP_ECONFIG, "null stage");
  const int dev = m0->cfg.device;
  int n_members = 0;
  for (int i = 0; i < n_items; ++i) {
    const tp_item& it = items[i];
    TP_CHECK(it.stage && it.stage->m->cfg.device == dev, TP_ECONFIG, "forward items must share one device");
    TP_CHECK(it.stage->m->cfg.arch == m0->cfg.arch, TP_ECONFIG, "forward items must share the arch");
    TP_CHECK(it.member >= 0 && it.member <= i, TP_ECONFIG, "member ids must be first-use ordered from 0");
    n_members = std::max(n_members, it.member + 1);
    for (int h = 0; h < i; ++h) TP_CHECK(items[h].stage != it.stage, TP_ECONFIG, "a stage appears twice");
  }
  TP_CUDA(cudaSetDevice(dev));
  cudaStream_t st = (cudaStream_t)stream;
  timeline_mark("host_gap", st);  // GPU time since the previous mark: idle or other work
  std::vector<LevelDev> lv(n_items);
  std::vector<size_t> off(n_items + 1, 0);
  std::vector<tp_level> tmp(n_items);
  std::vector<LevelStore> store(n_items);
  std::vector<const tp_level*> lvl(n_items);
  for (int i = 0; i < n_items; ++i) {
    lvl[i] = materialize(&items[i].level, &tmp[i], &store[i]);
    size_t b;
    TP_TRY(level_validate(items[i].stage, lvl[i], items[i].hidden_in, member_hidden_out[items[i].member], &lv[i],
                          &b));
    off[i + 1] = off[i] + b;
  }
  {  // every item's metadata in one upload
    char *h, *dm;
    int slot;
    TP_TRY(call_slot(m0, off[n_items], &h, &dm, &slot));
    for (int i = 0; i < n_items; ++i) level_write(lvl[i], &lv[i], h + off[i], dm + off[i]);
    TP_TRY(call_push(m0, slot, off[n_items], st));
  }
  if (is_toy(m0)) {
    TP_CHECK(n_members == n_items, TP_ECONFIG, "toy arch: one item per member");
    for (int i = 0; i < n_items; ++i)
      TP_TRY(toy_forward(items[i].stage, lv[i], items[i].hidden_in, member_hidden_out[items[i].member], st));
  } else {
    std::vector<std::vector<FwdItem>> per(n_members);
    for (int i = 0; i < n_items; ++i)
      per[items[i].member].push_back(FwdItem{items[i].stage, lv[i], items[i].hidden_in});
    std::vector<FwdMember> mem(n_members);
    for (int g = 0; g < n_members; ++g)
      mem[g] = FwdMember{per[g].data(), (int)per[g].size(), (float*)member_hidden_out[g]};
    for (int g0 = 0; g0 < n_members; g0 += kMaxGroup)
      TP_TRY(llama_forward_members(mem.data() + g0, std::min(kMaxGroup, n_members - g0), st, ws_base));
  }
  for (int i = 0; i < n_items; ++i)
    if (items[i].level.append) items[i].stage->rows += items[i].level.n;
  return TP_OK;
}

int tp_model_greedy_rows_async(tp_model* m, tp_stage* ws, int32_t n, const void* hidden_dev, void* stream) {
  TP_CUDA(cudaSetDevice(m->cfg.device));
  TP_CHECK(!is_toy(m), TP_ECONFIG, "multi-row verify is the llama path");
  TP_CHECK(ws && ws->m == m, TP_ECONFIG, "workspace stage must belong to the model");
  TP_CHECK(n >= 1 && n <= m->cfg.max_nodes, TP_ESHAPE, "rows outside [1, max_nodes]");
  if (ws->logits_rows < n) {
    TP_CUDA(cudaDeviceSynchronize());
    if (ws->logits) cudaFree(ws->logits);
    TP_CUDA(cudaMalloc(&ws->logits, (size_t)m->cfg.vocab * 8 * n));
    ws->logits_rows = n;
  }
  TP_TRY(llama_greedy_rows_async(m, n, (const float*)hidden_dev, (float*)ws->logits, (cudaStream_t)stream));
  count_io(0, 4LL * n);
  return TP_OK;
}

int tp_model_greedy_rows_wait(tp_model* m, int32_t n, int32_t* tokens_host) {
  TP_CUDA(cudaSetDevice(m->cfg.device));
  return llama_greedy_rows_wait(m, n, tokens_host);
}

int tp_stage_compact(tp_stage* s, int32_t first_row, int32_t count, const uint64_t* keep_bits, void* stream) {
  TP_CUDA(cudaSetDevice(s->m->cfg.device));
  TP_CHECK(first_row >= 0 && count >= 0 && first_row + count <= s->rows, TP_ECONTRACT,
           "compaction window outside the cache (prefix rows cannot be dropped)");
  std::vector<int32_t> src;
  src.reserve(count);
  for (int j = 0; j < count; ++j)
    if ((keep_bits[j >> 6] >> (j & 63)) & 1ull) src.push_back(first_row + j);
  if (!src.empty()) {
    cudaStream_t st = (cudaStream_t)stream;
    const char* d;
    TP_TRY(upload(s, src.data(), src.size() * 4, st, &d));
    TP_TRY(kv_compact(s, (const int32_t*)d, (int)src.size(), first_row, st));
    timeline_mark("kv_compact", st);
  }
  s->rows = first_row + (int)src.size();
  return TP_OK;
}

int tp_stages_compact(int32_t count, tp_stage* const* stages, const int32_t* first_rows, const int32_t* counts,
                      const uint64_t* const* keep_bits, void* stream) {
  TP_CHECK(count >= 0 && (count == 0 || (stages && first_rows && counts && keep_bits)), TP_ECONFIG, "null argument");
  if (count == 0) return TP_OK;
  tp_model* m0 = stages[0]->m;
  TP_CUDA(cudaSetDevice(m0->cfg.device));
  cudaStream_t st = (cudaStream_t)stream;
  for (int i = 0; i < count; ++i) {
    tp_stage* s = stages[i];
    TP_CHECK(s && s->m->cfg.device == m0->cfg.device, TP_ECONFIG, "stages of one compaction call share a device");
    TP_CHECK(first_rows[i] >= 0 && counts[i] >= 0 && first_rows[i] + counts[i] <= s->rows, TP_ECONTRACT,
             "compaction window outside the cache (prefix rows cannot be dropped)");
    TP_CHECK((s->head_dim * s->esize) % 16 == 0, TP_ESHAPE, "KV row bytes must be a multiple of 16");
  }
  for (int c0 = 0; c0 < count; c0 += kMaxMulti) {  // <= 64 stages per upload + launch
    const int c1 = std::min(count, c0 + kMaxMulti);
    std::vector<std::vector<int32_t>> src(c1 - c0);
    size_t bytes = 0;
    for (int i = c0; i < c1; ++i) {
      for (int j = 0; j < counts[i]; ++j)
        if ((keep_bits[i][j >> 6] >> (j & 63)) & 1ull) src[i - c0].push_back(first_rows[i] + j);
      bytes += (4 * src[i - c0].size() + 15) & ~(size_t)15;
    }
    char *h, *dm;
    int slot;
    TP_TRY(call_slot(m0, bytes, &h, &dm, &slot));
    MoveGroup g;
    g.count = 0;
    int ctas = 0;
    size_t off = 0;
    for (int i = c0; i < c1; ++i) {
      tp_stage* s = stages[i];
      const std::vector<int32_t>& v = src[i - c0];
      const int nl = s->hi - s->lo;
      std::memcpy(h + off, v.data(), 4 * v.size());
      if (!v.empty() && nl > 0) {
        MoveItem& it = g.m[g.count++];
        it.kv = kv_view(s);
        it.src = reinterpret_cast<const int32_t*>(dm + off);
        it.n_keep = (int)v.size();
        it.first = first_rows[i];
        it.cta0 = ctas;
        ctas += 2 * nl * s->kv_heads;
      }
      off += (4 * v.size() + 15) & ~(size_t)15;
      s->rows = first_rows[i] + (int)v.size();
    }
    TP_TRY(call_push(m0, slot, bytes, st));
    TP_TRY(kv_compact_many(g, ctas, st));
  }
  timeline_mark("kv_compact", st);
  return TP_OK;
}

int tp_rows_compact_many(int32_t count, tp_stage* ws, const void* const* src_dev, void* const* dst_dev,
                         int64_t row_bytes, const int32_t* n_src, const uint64_t* const* keep_bits, int32_t* n_out,
                         void* stream) {
  TP_CHECK(count >= 0 && count <= kMaxMulti && ws, TP_ECONFIG, "rows_compact_many: 0..64 sets and a workspace");
  if (count == 0) return TP_OK;
  TP_CUDA(cudaSetDevice(ws->m->cfg.device));
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<std::vector<int32_t>> idx(count);
  size_t bytes = 0;
  for (int i = 0; i < count; ++i) {
    for (int j = 0; j < n_src[i]; ++j)
      if ((keep_bits[i][j >> 6] >> (j & 63)) & 1ull) idx[i].push_back(j);
    n_out[i] = (int32_t)idx[i].size();
    bytes += (4 * idx[i].size() + 15) & ~(size_t)15;
  }
  char *h, *dm;
  int slot;
  TP_TRY(call_slot(ws->m, bytes, &h, &dm, &slot));
  RowsGroup g;
  g.count = 0;
  g.row_bytes = (int)row_bytes;
  size_t off = 0;
  int mr = 0;
  for (int i = 0; i < count; ++i) {
    std::memcpy(h + off, idx[i].data(), 4 * idx[i].size());
    if (!idx[i].empty()) {
      g.m[g.count++] = RowsItem{src_dev[i], dst_dev[i], reinterpret_cast<const int32_t*>(dm + off), n_out[i]};
      mr = std::max(mr, n_out[i]);
    }
    off += (4 * idx[i].size() + 15) & ~(size_t)15;
  }
  TP_TRY(call_push(ws->m, slot, bytes, st));
  TP_TRY(rows_compact_many(g, mr, st));
  timeline_mark("rows_compact", st);
  return TP_OK;
}

int tp_stage_truncate(tp_stage* s, int32_t rows) {
  TP_CHECK(rows >= 0 && rows <= s->rows, TP_ECONTRACT, "truncate beyond filled rows");
  s->rows = rows;
  return TP_OK;
}

int tp_stage_read_kv(const tp_stage* s, int32_t layer, int32_t kind, int32_t lo, int32_t hi, void* host) {
  TP_CUDA(cudaSetDevice(s->m->cfg.device));
  TP_CHECK(layer >= s->lo && layer < s->hi, TP_ESHAPE, "layer not hosted by stage");
  TP_CHECK(0 <= lo && lo <= hi && hi <= s->cap, TP_ESHAPE, "row range outside capacity");
  if (hi == lo) return TP_OK;
  size_t row = (size_t)s->head_dim * s->esize;
  TP_CUDA(cudaDeviceSynchronize());
  if (!is_toy(s->m)) {  // paged: gather on the device, one copy out
    void* d = nullptr;
    const size_t bytes = (size_t)(hi - lo) * s->kv_heads * row;
    TP_CUDA(cudaMalloc(&d, bytes));
    int rc = kv_read_rows(s, layer, kind, lo, hi, d, 0);
    if (rc == TP_OK) TP_CUDA(cudaMemcpy(host, d, bytes, cudaMemcpyDeviceToHost));
    cudaFree(d);
    return rc;
  }
  const char* plane = (const char*)(kind == 0 ? s->k : s->v)[layer - s->lo];
  for (int h = 0; h < s->kv_heads; ++h)
    TP_CUDA(cudaMemcpy2D((char*)host + h * row, row * s->kv_heads, plane + (h * (size_t)s->cap + lo) * row, row,
                         row, hi - lo, cudaMemcpyDeviceToHost));
  return TP_OK;
}

int tp_model_embed(tp_model* m, int32_t n, const int32_t* tokens, const int32_t* positions, void* out_dev,
                   void* stream) {
  // uses a transient stage-free path: small synchronous upload
  TP_CUDA(cudaSetDevice(m->cfg.device));
  TP_CHECK(m->embed, TP_ECONFIG, "model has no embedding table");
  for (int i = 0; i < n; ++i) TP_CHECK(tokens[i] >= 0 && tokens[i] < m->cfg.vocab, TP_ESHAPE, "token outside vocabulary");
  int32_t* d = nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  TP_CUDA(cudaMallocAsync((void**)&d, 8 * (size_t)n, st));
  TP_CUDA(cudaMemcpyAsync(d, tokens, 4 * (size_t)n, cudaMemcpyHostToDevice, st));
  TP_CUDA(cudaMemcpyAsync(d + n, positions, 4 * (size_t)n, cudaMemcpyHostToDevice, st));
  int rc = is_toy(m) ? toy_embed(m, n, d, d + n, (double*)out_dev, st) : llama_embed(m, n, d, (float*)out_dev, st);
  cudaFreeAsync(d, st);
  return rc;
}

int tp_model_logits(tp_model* m, tp_stage* ws, int32_t n, const void* hidden_dev, void* logits_dev, void* stream) {
  TP_CUDA(cudaSetDevice(m->cfg.device));
  TP_CHECK(ws && ws->m == m, TP_ECONFIG, "workspace stage must belong to the model");
  TP_CHECK(n >= 1 && n <= m->cfg.max_nodes, TP_ESHAPE, "rows outside [1, max_nodes]");
  cudaStream_t st = (cudaStream_t)stream;
  return is_toy(m) ? toy_logits(m, ws, n, (const double*)hidden_dev, (double*)logits_dev, st)
                   : llama_logits(m, ws, n, (const float*)hidden_dev, (float*)logits_dev, st);
}

int tp_model_verify_async(tp_model* m, tp_stage* ws, const void* hidden_dev, const int32_t* child_tokens,
                          int32_t n_children, void* stream) {
  TP_CUDA(cudaSetDevice(m->cfg.device));
  TP_CHECK(ws && ws->m == m, TP_ECONFIG, "workspace stage must belong to the model");
  TP_CHECK(n_children >= 0 && n_children <= m->cfg.max_nodes, TP_ESHAPE, "too many children");
  cudaStream_t st = (cudaStream_t)stream;
  TP_TRY(tp_model_logits(m, ws, 1, hidden_dev, ws->logits, stream));
  const char* d = nullptr;
  if (n_children) TP_TRY(upload(ws, child_tokens, 4 * (size_t)n_children, st, &d));
  TP_TRY(argmax_match(ws->logits, is_toy(m), m->cfg.vocab, (const int32_t*)d, n_children, ws->d_result, st));
  TP_CUDA(cudaMemcpyAsync(ws->h_result, ws->d_result, 8, cudaMemcpyDeviceToHost, st));
  count_io(0, 8);
  timeline_mark("verify_head", st);
  TP_CUDA(cudaEventRecord(ws->verify_ev, st));
  return TP_OK;
}

int tp_model_verify_wait(tp_stage* ws, int32_t* result_host) {
  TP_CHECK(ws, TP_ECONFIG, "null argument");
  TP_CUDA(cudaEventSynchronize(ws->verify_ev));
  result_host[0] = ws->h_result[0];
  result_host[1] = ws->h_result[1];
  return TP_OK;
}

int tp_model_verify(tp_model* m, tp_stage* ws, const void* hidden_dev, const int32_t* child_tokens,
                    int32_t n_children, int32_t* result_host, void* stream) {
  TP_TRY(tp_model_verify_async(m, ws, hidden_dev, child_tokens, n_children, stream));
  return tp_model_verify_wait(ws, result_host);
}

int tp_rows_compact(tp_stage* ws, const void* src_dev, void* dst_dev, int64_t row_bytes, int32_t n_src,
                    const uint64_t* keep_bits, int32_t* n_out, void* stream) {
  TP_CUDA(cudaSetDevice(ws->m->cfg.device));
  std::vector<int32_t> idx;
  for (int j = 0; j < n_src; ++j)
    if ((keep_bits[j >> 6] >> (j & 63)) & 1ull) idx.push_back(j);
  *n_out = (int32_t)idx.size();
  if (idx.empty()) return TP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const char* d;
  TP_TRY(upload(ws, idx.data(), idx.size() * 4, st, &d));
  TP_TRY(rows_compact(src_dev, dst_dev, row_bytes, (const int32_t*)d, (int)idx.size(), st));
  timeline_mark("rows_compact", st);
  return TP_OK;
}

}  // extern "C"
