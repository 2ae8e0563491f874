// memexec.cu — Host tier (pinned FixedBufferPool) and Device<->Host moves of
// chunked batches (include/tq_memexec.h).  Layout rules follow the
// reference's encode_chunked / decode_chunked (chunked.cpp:19-118): sections
// (values, validity, offsets per column, in schema order) laid end to end
// across pool buffers; section lengths validated against the schema.
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <vector>

#include "../../include/tq_memexec.h"
#include "ctx.h"
#include "memexec_internal.h"

namespace tq {
namespace {

// section sizes of a batch: values, validity, offsets (types.cpp:146-164)
std::vector<uint64_t> section_sizes(const tq_batch* b) {
  std::vector<uint64_t> s;
  for (uint32_t c = 0; c < b->ncols; ++c) {
    const tq_column& col = b->cols[c];
    s.push_back(col.values_bytes);
    s.push_back(col.validity && b->rows ? (b->rows + 7) / 8 : 0);
    s.push_back(col.kind == TQ_UTF8 ? (b->rows + 1) * 4 : 0);
  }
  return s;
}

std::vector<uint32_t> acquire(tq_pool* p, uint64_t n) {
  std::lock_guard<std::mutex> g(p->mu);
  if (p->free_list.size() < n) fail(TQ_POOL_EXHAUSTED, "pinned pool exhausted");
  std::vector<uint32_t> ids;
  ids.reserve(n);
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t id = p->free_list.back();
    p->free_list.pop_back();
    p->in_use[id] = true;
    ids.push_back(id);
  }
  return ids;
}

void release(tq_pool* p, const uint32_t* ids, uint64_t n) {
  std::lock_guard<std::mutex> g(p->mu);
  for (uint64_t i = 0; i < n; ++i) {
    if (ids[i] >= p->capacity) fail(TQ_INTERNAL, "release of unknown buffer id");
    if (!p->in_use[ids[i]]) fail(TQ_INTERNAL, "double release of buffer");
  }
  for (uint64_t i = 0; i < n; ++i) {
    p->in_use[ids[i]] = false;
    p->free_list.push_back(ids[i]);
  }
}

// Lay out `sizes` across freshly acquired buffers (encode_chunked's layout).
tq_chunked* layout(tq_pool* pool, const tq_batch* b) {
  auto sizes = section_sizes(b);
  uint64_t total = std::accumulate(sizes.begin(), sizes.end(), 0ull);
  const uint64_t bs = pool->buffer_size;
  const uint64_t nbuf = bs ? (total + bs - 1) / bs : 0;
  tq_chunked* cb = new tq_chunked();
  cb->pool = pool;
  cb->rows = b->rows;
  cb->total = total;
  cb->tail = nbuf * bs - total;
  for (uint32_t c = 0; c < b->ncols; ++c) {
    tq_column s{};
    s.kind = b->cols[c].kind;
    s.precision = b->cols[c].precision;
    s.scale = b->cols[c].scale;
    cb->schema.push_back(s);
  }
  try {
    if (nbuf) cb->buffers = acquire(pool, nbuf);
  } catch (...) {
    delete cb;
    throw;
  }
  uint64_t cursor = 0;
  for (uint64_t len : sizes) {
    cb->sec_len.push_back(len);
    std::vector<Seg> segs;
    uint64_t done = 0;
    while (done < len) {
      uint32_t buf = cb->buffers[cursor / bs];
      uint64_t in = cursor % bs;
      uint64_t take = std::min<uint64_t>(bs - in, len - done);
      segs.push_back({buf, (uint32_t)in, (uint32_t)take});
      done += take;
      cursor += take;
    }
    cb->sec_segs.push_back(std::move(segs));
  }
  return cb;
}

const uint8_t* sec_ptr(const tq_column& col, int part, uint64_t rows) {
  if (part == 0) return (const uint8_t*)col.values;
  if (part == 1) return rows ? col.validity : nullptr;
  return (const uint8_t*)col.offsets;
}

// schema-derived section length checks (section_fixed_length, types.cpp:172-184)
void validate(const tq_chunked* cb) {
  if (cb->sec_len.size() != cb->schema.size() * 3) fail(TQ_CORRUPT_LAYOUT, "section count disagrees with schema");
  for (size_t c = 0; c < cb->schema.size(); ++c) {
    const tq_column& s = cb->schema[c];
    uint64_t vlen = cb->sec_len[c * 3], blen = cb->sec_len[c * 3 + 1], olen = cb->sec_len[c * 3 + 2];
    bool hv = blen > 0;
    if (hv && blen != (cb->rows + 7) / 8) fail(TQ_CORRUPT_LAYOUT, "validity length disagrees with schema");
    if (s.kind == TQ_UTF8) {
      if (olen != (cb->rows + 1) * 4) fail(TQ_CORRUPT_LAYOUT, "offsets length disagrees with schema");
    } else {
      if (olen != 0) fail(TQ_CORRUPT_LAYOUT, "offsets on fixed-width column");
      if (vlen != cb->rows * width_of(s.kind)) fail(TQ_CORRUPT_LAYOUT, "values length disagrees with schema");
    }
    for (int part = 0; part < 3; ++part) {
      uint64_t sum = 0;
      for (const Seg& g : cb->sec_segs[c * 3 + part]) {
        if ((uint64_t)g.off + g.len > cb->pool->buffer_size) fail(TQ_CORRUPT_LAYOUT, "segment exceeds buffer bounds");
        sum += g.len;
      }
      if (sum != cb->sec_len[c * 3 + part]) fail(TQ_CORRUPT_LAYOUT, "segment lengths disagree with section length");
    }
  }
}

}  // namespace

tq_chunked* chunked_layout(tq_pool* pool, const tq_batch* b) { return layout(pool, b); }

}  // namespace tq

using namespace tq;

extern "C" {

tq_status tq_pool_create(uint64_t buffer_size, uint64_t capacity, tq_pool** out) {
  return guard([&] {
    if (buffer_size == 0) fail(TQ_INTERNAL, "buffer_size must be positive");
    tq_pool* p = new tq_pool();
    p->buffer_size = buffer_size;
    p->capacity = capacity;
    if (capacity) {
      cudaError_t e = cudaHostAlloc((void**)&p->arena, buffer_size * capacity, cudaHostAllocPortable);
      if (e != cudaSuccess) {
        cudaGetLastError();
        // no driver (CPU-only box): plain host memory keeps the tier usable for tests
        p->arena = (uint8_t*)std::malloc(buffer_size * capacity);
        if (!p->arena) {
          delete p;
          fail(TQ_POOL_EXHAUSTED, "cannot allocate host pool");
        }
      }
    }
    p->free_list.resize(capacity);
    std::iota(p->free_list.rbegin(), p->free_list.rend(), 0u);  // hand out low ids first
    p->in_use.assign(capacity, false);
    *out = p;
  });
}

void tq_pool_destroy(tq_pool* p) {
  if (!p) return;
  if (p->arena && cudaFreeHost(p->arena) != cudaSuccess) {
    cudaGetLastError();
    std::free(p->arena);
  }
  delete p;
}

uint64_t tq_pool_free_count(tq_pool* p) {
  std::lock_guard<std::mutex> g(p->mu);
  return p->free_list.size();
}
uint64_t tq_pool_buffer_size(tq_pool* p) { return p->buffer_size; }

tq_status tq_pool_acquire(tq_pool* p, uint64_t n, uint32_t* ids) {
  return guard([&] {
    if (n == 0) fail(TQ_INTERNAL, "acquire of zero buffers");
    auto v = acquire(p, n);
    std::memcpy(ids, v.data(), n * 4);
  });
}
tq_status tq_pool_release(tq_pool* p, const uint32_t* ids, uint64_t n) {
  return guard([&] { release(p, ids, n); });
}
uint8_t* tq_pool_buffer(tq_pool* p, uint32_t id) { return p->arena + (uint64_t)id * p->buffer_size; }

tq_status tq_chunked_encode(tq_pool* pool, const tq_batch* b, tq_chunked** out) {
  return guard([&] {
    if (b->mem != TQ_MEM_HOST) fail(TQ_INTERNAL, "tq_chunked_encode needs a host batch");
    tq_chunked* cb = layout(pool, b);
    for (uint32_t c = 0; c < b->ncols; ++c)
      for (int part = 0; part < 3; ++part) {
        const uint8_t* src = sec_ptr(b->cols[c], part, b->rows);
        uint64_t done = 0;
        for (const Seg& g : cb->sec_segs[c * 3 + part]) {
          std::memcpy(tq_pool_buffer(pool, g.buf) + g.off, src + done, g.len);
          done += g.len;
        }
      }
    *out = cb;
  });
}

tq_status tq_chunked_decode(const tq_chunked* cb, tq_batch* out) {
  return guard([&] {
    validate(cb);
    out->rows = cb->rows;
    out->ncols = (uint32_t)cb->schema.size();
    out->mem = TQ_MEM_HOST;
    out->owner = nullptr;
    out->cols = (tq_column*)std::calloc(std::max<size_t>(1, cb->schema.size()), sizeof(tq_column));
    for (size_t c = 0; c < cb->schema.size(); ++c) {
      tq_column& d = out->cols[c];
      d = cb->schema[c];
      d.values_bytes = cb->sec_len[c * 3];
      for (int part = 0; part < 3; ++part) {
        uint64_t len = cb->sec_len[c * 3 + part];
        if (part > 0 && len == 0) continue;
        uint8_t* dst = (uint8_t*)std::malloc(len ? len : 1);
        uint64_t done = 0;
        for (const Seg& g : cb->sec_segs[c * 3 + part]) {
          std::memcpy(dst + done, tq_pool_buffer(cb->pool, g.buf) + g.off, g.len);
          done += g.len;
        }
        if (part == 0) d.values = dst;
        else if (part == 1) d.validity = dst;
        else d.offsets = (int32_t*)dst;
      }
    }
  });
}

tq_status tq_spill(tq_ctx* c, tq_pool* pool, const tq_batch* dev, tq_chunked** out, void* stream) {
  return guard([&] {
    if (dev->mem != TQ_MEM_DEVICE) fail(TQ_INTERNAL, "tq_spill needs a device batch");
    cudaStream_t st = pick(c, stream);
    tq_chunked* cb = layout(pool, dev);
    for (uint32_t k = 0; k < dev->ncols; ++k)
      for (int part = 0; part < 3; ++part) {
        const uint8_t* src = sec_ptr(dev->cols[k], part, dev->rows);
        uint64_t done = 0;
        for (const Seg& g : cb->sec_segs[k * 3 + part]) {
          TQ_CUDA(cudaMemcpyAsync(tq_pool_buffer(pool, g.buf) + g.off, src + done, g.len, cudaMemcpyDeviceToHost, st));
          done += g.len;
        }
      }
    *out = cb;
  });
}

tq_status tq_load(tq_ctx* c, const tq_chunked* cb, tq_batch* out, void* stream) {
  return guard([&] {
    validate(cb);
    cudaStream_t st = pick(c, stream);
    std::vector<bool> wv;
    std::vector<uint64_t> ub;
    for (size_t k = 0; k < cb->schema.size(); ++k) {
      wv.push_back(cb->sec_len[k * 3 + 1] > 0);
      ub.push_back(cb->sec_len[k * 3]);
    }
    alloc_batch(c, cb->rows, cb->schema, wv, out, st, &ub);
    for (size_t k = 0; k < cb->schema.size(); ++k)
      for (int part = 0; part < 3; ++part) {
        uint8_t* dst = part == 0 ? (uint8_t*)out->cols[k].values
                                 : part == 1 ? out->cols[k].validity : (uint8_t*)out->cols[k].offsets;
        uint64_t done = 0;
        for (const Seg& g : cb->sec_segs[k * 3 + part]) {
          TQ_CUDA(cudaMemcpyAsync(dst + done, tq_pool_buffer(cb->pool, g.buf) + g.off, g.len, cudaMemcpyHostToDevice, st));
          done += g.len;
        }
      }
  });
}

uint32_t tq_chunked_layout(const tq_chunked* cb, uint64_t* nbuf, uint64_t* tail, uint64_t* total, uint32_t* segs,
                           uint32_t cap) {
  if (nbuf) *nbuf = cb->buffers.size();
  if (tail) *tail = cb->tail;
  if (total) *total = cb->total;
  uint32_t k = 0;
  for (const auto& v : cb->sec_segs)
    for (const Seg& g : v) {
      if (segs && k < cap) {
        segs[3 * k] = g.buf;
        segs[3 * k + 1] = g.off;
        segs[3 * k + 2] = g.len;
      }
      ++k;
    }
  return k;
}

uint64_t tq_chunked_rows(const tq_chunked* cb) { return cb->rows; }

void tq_chunked_release(tq_chunked* cb) {
  if (!cb) return;
  try {
    if (!cb->buffers.empty()) release(cb->pool, cb->buffers.data(), cb->buffers.size());
  } catch (...) {
  }
  delete cb;
}

}  // extern "C"
