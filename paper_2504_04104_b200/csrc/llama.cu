// Llama-arch stage compute (placeholder until the tcgen05 path lands).
#include "internal.h"

namespace tp {
int llama_forward(tp_stage*, const LevelDev&, const void*, void*, cudaStream_t) {
  set_error("llama path not implemented yet");
  return TP_ECONFIG;
}
int llama_embed(tp_model*, int, const int32_t*, float*, cudaStream_t) { set_error("llama: n/a"); return TP_ECONFIG; }
int llama_logits(tp_model*, tp_stage*, int, const float*, float*, cudaStream_t) { set_error("llama: n/a"); return TP_ECONFIG; }
int llama_workspace_bytes(const tp_model*, int, size_t* b) { *b = 256; return TP_OK; }
int llama_init_weights(tp_model*, uint64_t, cudaStream_t) { set_error("llama: n/a"); return TP_ECONFIG; }
}  // namespace tp
