// memexec_internal.h — the Host tier's pool / chunked-batch structures,
// shared by memexec.cu (spill / load) and storage.cu (TCF byte-range fetches
// straight into pool buffers).
#pragma once
#include <cstdint>
#include <mutex>
#include <vector>

#include "../../include/tq_memexec.h"

struct tq_pool {
  uint64_t buffer_size = 0, capacity = 0;
  uint8_t* arena = nullptr;  // cudaHostAlloc(portable): one allocation, never grown
  std::mutex mu;
  std::vector<uint32_t> free_list;  // LIFO; low ids first
  std::vector<bool> in_use;
};

struct Seg {
  uint32_t buf, off, len;
};
struct tq_chunked {
  tq_pool* pool = nullptr;
  uint64_t rows = 0;
  std::vector<tq_column> schema;           // kind / precision / scale (pointers unused)
  std::vector<uint64_t> sec_len;           // 3 per column
  std::vector<std::vector<Seg>> sec_segs;  // 3 per column
  std::vector<uint32_t> buffers;
  uint64_t total = 0, tail = 0;
};


namespace tq {
// Lay out a batch's sections (values, validity, offsets per column; only the
// section SIZES of `b` are read) across freshly acquired pool buffers.
tq_chunked* chunked_layout(tq_pool* pool, const tq_batch* b);
}  // namespace tq
