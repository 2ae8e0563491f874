// storage.cu — TCF files and their byte-range preload into the pinned Host
// pool (include/tq_storage.h; SPEC.md:128-229 storage module).
// Host code: POSIX pread for the LocalDisk datasource, reads issued
// concurrently up to the connection limit, straight into the pool buffers of
// a chunked batch that tq_load then moves to the device.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/tq_storage.h"
#include "ctx.h"
#include "memexec_internal.h"

namespace {
using namespace tq;

constexpr char kMagic[4] = {'T', 'C', 'F', '1'};

struct ColMeta {
  uint64_t offset, values_len, validity_len, offsets_len;
  uint64_t length() const { return values_len + validity_len + offsets_len; }
};
struct RowGroup {
  uint64_t rows;
  std::vector<ColMeta> cols;
};

void put(std::string& b, const void* p, size_t n) { b.append((const char*)p, n); }
template <class T>
void put(std::string& b, T v) {
  put(b, &v, sizeof v);
}

struct Reader {  // bounds-checked footer parsing (CorruptFooter)
  const uint8_t* p;
  size_t n, at = 0;
  void get(void* d, size_t k) {
    if (at + k > n) fail(TQ_CORRUPT_FOOTER, "TCF footer truncated");
    std::memcpy(d, p + at, k);
    at += k;
  }
  template <class T>
  T get() {
    T v;
    get(&v, sizeof v);
    return v;
  }
};

void pread_all(int fd, void* dst, uint64_t len, uint64_t off) {
  uint8_t* d = (uint8_t*)dst;
  while (len) {
    const ssize_t r = ::pread(fd, d, len, (off_t)off);
    if (r <= 0) fail(TQ_IO_ERROR, "TCF read failed");
    d += r;
    off += (uint64_t)r;
    len -= (uint64_t)r;
  }
}

}  // namespace

struct tq_tcf {
  int fd = -1;
  uint64_t size = 0;
  std::vector<tq_column> schema;
  std::vector<std::string> names;
  std::vector<RowGroup> rgs;
  std::atomic<uint64_t> reads{0};
  void read(void* dst, uint64_t len, uint64_t off) {
    reads++;
    pread_all(fd, dst, len, off);
  }
};

extern "C" {

tq_status tq_tcf_write(const char* path, const tq_batch* t, const char* const* names, uint64_t rg_bytes) {
  return guard([&] {
    if (t->mem != TQ_MEM_HOST) fail(TQ_INTERNAL, "tq_tcf_write takes a host batch");
    if (rg_bytes == 0) fail(TQ_INTERNAL, "row group target must be positive");
    uint64_t total = 0;
    for (uint32_t c = 0; c < t->ncols; ++c) {
      const tq_column& col = t->cols[c];
      total += col.values_bytes + (col.validity && t->rows ? (t->rows + 7) / 8 : 0) +
               (col.kind == TQ_UTF8 ? (t->rows + 1) * 4 : 0);
    }
    // rows per group: the target over the average row, a multiple of 8 so a
    // group's bitmap is a byte range of the column's
    uint64_t per = t->rows ? std::max<uint64_t>(8, (uint64_t)((double)rg_bytes * t->rows / std::max<uint64_t>(1, total))) : 0;
    per = per / 8 * 8;
    std::string file(kMagic, 4), footer;
    std::vector<RowGroup> rgs;
    for (uint64_t r0 = 0; r0 < t->rows; r0 += per) {
      const uint64_t n = std::min(per, t->rows - r0);
      RowGroup rg{n, {}};
      for (uint32_t c = 0; c < t->ncols; ++c) {
        const tq_column& col = t->cols[c];
        ColMeta m{file.size(), 0, 0, 0};
        if (col.kind == TQ_UTF8) {
          const int32_t a = col.offsets[r0], e = col.offsets[r0 + n];
          put(file, (const uint8_t*)col.values + a, (size_t)(e - a));
          m.values_len = (uint64_t)(e - a);
        } else {
          const uint64_t w = width_of(col.kind);
          put(file, (const uint8_t*)col.values + r0 * w, n * w);
          m.values_len = n * w;
        }
        if (col.validity) {
          std::string bm((n + 7) / 8, '\0');
          std::memcpy(&bm[0], col.validity + r0 / 8, bm.size());
          if (n % 8) bm.back() &= (char)((1u << (n % 8)) - 1);  // padding bits zero (types.cpp:123-131)
          file += bm;
          m.validity_len = bm.size();
        }
        if (col.kind == TQ_UTF8) {  // rebased to the group's first string
          const int32_t base = col.offsets[r0];
          for (uint64_t i = 0; i <= n; ++i) put<int32_t>(file, col.offsets[r0 + i] - base);
          m.offsets_len = (n + 1) * 4;
        }
        rg.cols.push_back(m);
      }
      rgs.push_back(rg);
    }
    put<uint32_t>(footer, t->ncols);
    for (uint32_t c = 0; c < t->ncols; ++c) {
      const std::string nm = names && names[c] ? names[c] : "c" + std::to_string(c);
      put<uint8_t>(footer, t->cols[c].kind);
      put<uint8_t>(footer, t->cols[c].precision);
      put<uint8_t>(footer, t->cols[c].scale);
      put<uint16_t>(footer, (uint16_t)nm.size());
      footer += nm;
    }
    put<uint32_t>(footer, (uint32_t)rgs.size());
    for (const RowGroup& rg : rgs) {
      put<uint64_t>(footer, rg.rows);
      for (const ColMeta& m : rg.cols) put(footer, &m, sizeof m);
    }
    file += footer;
    put<uint32_t>(file, (uint32_t)footer.size());
    file.append(kMagic, 4);
    const int fd = ::open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (fd < 0) fail(TQ_IO_ERROR, std::string("cannot create ") + path);
    size_t done = 0;
    while (done < file.size()) {
      const ssize_t w = ::write(fd, file.data() + done, file.size() - done);
      if (w <= 0) {
        ::close(fd);
        fail(TQ_IO_ERROR, "TCF write failed");
      }
      done += (size_t)w;
    }
    ::close(fd);
  });
}

tq_status tq_tcf_open(const char* path, tq_tcf** out) {
  return guard([&] {
    tq_tcf* f = new tq_tcf();
    try {
      f->fd = ::open(path, O_RDONLY);
      if (f->fd < 0) fail(TQ_IO_ERROR, std::string("cannot open ") + path);
      struct stat st;
      if (::fstat(f->fd, &st) != 0) fail(TQ_IO_ERROR, "fstat failed");
      f->size = (uint64_t)st.st_size;
      if (f->size < 12) fail(TQ_NOT_TCF, "file too small for TCF");
      // read_footer: exactly two reads — the trailing length + magic, then the footer
      uint8_t tail[8];
      f->read(tail, 8, f->size - 8);
      if (std::memcmp(tail + 4, kMagic, 4) != 0) fail(TQ_NOT_TCF, "missing TCF trailing magic");
      uint32_t flen;
      std::memcpy(&flen, tail, 4);
      if ((uint64_t)flen + 12 > f->size) fail(TQ_CORRUPT_FOOTER, "footer length exceeds file");
      std::vector<uint8_t> fb(flen);
      f->read(fb.data(), flen, f->size - 8 - flen);
      Reader r{fb.data(), fb.size()};
      const uint32_t ncols = r.get<uint32_t>();
      for (uint32_t c = 0; c < ncols; ++c) {
        tq_column col{};
        col.kind = r.get<uint8_t>();
        col.precision = r.get<uint8_t>();
        col.scale = r.get<uint8_t>();
        if (col.kind > TQ_DECIMAL) fail(TQ_CORRUPT_FOOTER, "bad column kind");
        std::string nm(r.get<uint16_t>(), '\0');
        if (!nm.empty()) r.get(&nm[0], nm.size());
        f->schema.push_back(col);
        f->names.push_back(nm);
      }
      const uint32_t nrg = r.get<uint32_t>();
      const uint64_t data_end = f->size - 8 - flen;
      uint64_t prev_end = 4;
      for (uint32_t g = 0; g < nrg; ++g) {
        RowGroup rg{r.get<uint64_t>(), {}};
        for (uint32_t c = 0; c < ncols; ++c) {
          ColMeta m;
          r.get(&m, sizeof m);
          // ranges within the file, ascending, non-overlapping (SPEC.md TcfFooter invariants)
          if (m.offset < prev_end || m.offset + m.length() > data_end) fail(TQ_CORRUPT_FOOTER, "column range out of order");
          prev_end = m.offset + m.length();
          rg.cols.push_back(m);
        }
        f->rgs.push_back(rg);
      }
    } catch (...) {
      tq_tcf_close(f);
      throw;
    }
    *out = f;
  });
}

void tq_tcf_close(tq_tcf* f) {
  if (!f) return;
  if (f->fd >= 0) ::close(f->fd);
  delete f;
}

uint32_t tq_tcf_ncols(const tq_tcf* f) { return (uint32_t)f->schema.size(); }
uint32_t tq_tcf_row_groups(const tq_tcf* f) { return (uint32_t)f->rgs.size(); }
uint64_t tq_tcf_rows(const tq_tcf* f, uint32_t g) { return g < f->rgs.size() ? f->rgs[g].rows : 0; }
uint64_t tq_tcf_reads(const tq_tcf* f) { return f->reads.load(); }

const char* tq_tcf_column(const tq_tcf* f, uint32_t c, tq_column* col) {
  if (c >= f->schema.size()) return nullptr;
  if (col) {
    col->kind = f->schema[c].kind;
    col->precision = f->schema[c].precision;
    col->scale = f->schema[c].scale;
  }
  return f->names[c].c_str();
}

tq_status tq_tcf_plan_ranges(const tq_tcf* f, const uint32_t* cols, uint32_t ncols, const uint32_t* rgs, uint32_t nrg,
                             tq_range* out, uint64_t cap, uint64_t* n) {
  return guard([&] {
    std::vector<tq_range> v;
    for (uint32_t i = 0; i < nrg; ++i) {
      if (rgs[i] >= f->rgs.size()) fail(TQ_CORRUPT_ROW_GROUP, "no such row group");
      for (uint32_t k = 0; k < ncols; ++k) {
        if (cols[k] >= f->schema.size()) fail(TQ_UNKNOWN_COLUMN, "no such column");
        const ColMeta& m = f->rgs[rgs[i]].cols[cols[k]];
        if (m.length()) v.push_back({m.offset, m.length()});
      }
    }
    std::sort(v.begin(), v.end(), [](const tq_range& a, const tq_range& b) { return a.offset < b.offset; });
    for (uint64_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
    *n = v.size();
  });
}

uint64_t tq_coalesce_ranges(const tq_range* in, uint64_t n, uint64_t max_gap, uint64_t max_merged, tq_range* out) {
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (k) {
      tq_range& last = out[k - 1];
      const uint64_t end = last.offset + last.length;
      const uint64_t merged = in[i].offset + in[i].length - last.offset;
      if (in[i].offset >= end && in[i].offset - end <= max_gap && merged <= max_merged) {
        last.length = merged;
        continue;
      }
    }
    out[k++] = in[i];
  }
  return k;
}

tq_status tq_tcf_fetch(tq_tcf* f, tq_pool* pool, uint32_t g, const uint32_t* cols, uint32_t ncols, uint32_t max_conn,
                       tq_chunked** out) {
  return guard([&] {
    if (g >= f->rgs.size()) fail(TQ_CORRUPT_ROW_GROUP, "no such row group");
    const RowGroup& rg = f->rgs[g];
    // a size-only descriptor of the needed columns: the chunked layout of their sections
    std::vector<tq_column> desc(ncols);
    static uint8_t nonnull;  // (validity presence only)
    for (uint32_t k = 0; k < ncols; ++k) {
      if (cols[k] >= f->schema.size()) fail(TQ_UNKNOWN_COLUMN, "no such column");
      const ColMeta& m = rg.cols[cols[k]];
      tq_column& d = desc[k];
      d = f->schema[cols[k]];
      d.values_bytes = m.values_len;
      d.validity = m.validity_len ? &nonnull : nullptr;
      const bool utf8 = d.kind == TQ_UTF8;
      if ((!utf8 && m.values_len != rg.rows * width_of(d.kind)) || (m.validity_len && m.validity_len != (rg.rows + 7) / 8) ||
          (utf8 && m.offsets_len != (rg.rows + 1) * 4) || (!utf8 && m.offsets_len))
        fail(TQ_CORRUPT_ROW_GROUP, "column section lengths disagree with the schema");
    }
    tq_batch d{rg.rows, ncols, TQ_MEM_HOST, desc.data(), nullptr};
    tq_chunked* cb = chunked_layout(pool, &d);
    // column k's file range [offset, offset + length) is the chunked byte
    // stream [cursor_k, cursor_k + length): split it at buffer boundaries
    struct Read {
      uint8_t* dst;
      uint64_t off, len;
    };
    std::vector<Read> reads;
    const uint64_t bs = pool->buffer_size;
    uint64_t cursor = 0;
    for (uint32_t k = 0; k < ncols; ++k) {
      const ColMeta& m = rg.cols[cols[k]];
      uint64_t done = 0;
      while (done < m.length()) {
        const uint64_t at = cursor + done;
        const uint64_t in = at % bs, take = std::min(bs - in, m.length() - done);
        uint8_t* dst = pool->arena + (uint64_t)cb->buffers[at / bs] * bs + in;
        // touching reads (the next column's bytes follow in the file and in the
        // pool buffer) are issued as one
        if (!reads.empty() && reads.back().off + reads.back().len == m.offset + done &&
            reads.back().dst + reads.back().len == dst)
          reads.back().len += take;
        else
          reads.push_back({dst, m.offset + done, take});
        done += take;
      }
      cursor += m.length();
    }
    // up to max_conn preads in flight (the datasource's connection limit)
    const uint32_t nt = std::max<uint32_t>(1, std::min<uint32_t>(max_conn ? max_conn : 4, (uint32_t)reads.size()));
    std::atomic<size_t> next{0};
    std::atomic<bool> bad{false};
    std::vector<std::thread> ts;
    for (uint32_t t = 0; t < nt; ++t)
      ts.emplace_back([&] {
        for (size_t i; (i = next.fetch_add(1)) < reads.size();) {
          try {
            f->read(reads[i].dst, reads[i].len, reads[i].off);
          } catch (...) {
            bad = true;
          }
        }
      });
    for (auto& t : ts) t.join();
    if (bad) {
      tq_chunked_release(cb);
      fail(TQ_IO_ERROR, "TCF range read failed");
    }
    *out = cb;
  });
}

}  // extern "C"
