// Workspace planning: collect every scratch buffer a call needs, reserve the
// arena once (the only place that may allocate), then hand out slices.
#pragma once

#include <vector>

#include "common.cuh"

namespace orchb {

class Plan {
 public:
  template <class T>
  void add(T** slot, size_t count) {
    const size_t bytes = count * sizeof(T);
    entries_.push_back({reinterpret_cast<void**>(slot), bytes});
    total_ += (bytes + 255) & ~size_t{255};
  }
  // Use the caller's buffer when given, else a workspace slice.
  template <class T>
  void add_or(T** slot, T* given, size_t count) {
    if (given) {
      *slot = given;
    } else {
      add(slot, count);
    }
  }
  int commit(orch_ctx* ctx, cudaStream_t stream) {
    Arena* a = arena_for(ctx, stream);
    if (!a) return fail(ORCH_CUDA_ERROR, "workspace hand-over to a new stream failed (device synchronisation)");
    int rc = arena_reserve(a, total_ + 256, stream);
    if (rc) return rc;
    a->used = 0;  // calls on one stream run in order: the previous call's scratch is free
    for (auto& e : entries_) {
      *e.slot = carve(a, e.bytes ? e.bytes : 1);
      if (!*e.slot) return fail(ORCH_CUDA_ERROR, "workspace arena exhausted");
    }
    return ORCH_OK;
  }
  size_t total() const { return total_; }

 private:
  struct Entry {
    void** slot;
    size_t bytes;
  };
  std::vector<Entry> entries_;
  size_t total_ = 0;
};

}  // namespace orchb
