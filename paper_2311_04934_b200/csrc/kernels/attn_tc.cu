// tcgen05 flash attention for the bf16 hot path (suffix queries over the
// assembled cache, and causal prefill).  Round-1 bring-up: not yet enabled —
// attention_tc_supported() returns false and the SIMT kernel runs.
#include "common.cuh"

namespace pcb::kern {
bool attention_tc_supported(const AttnArgs&) { return false; }
void attention_tc(const AttnArgs&, float*, size_t, cudaStream_t) {
  throw std::runtime_error("attention_tc not available");
}
}  // namespace pcb::kern
