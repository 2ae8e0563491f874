// exchange.cu — the shuffle (include/tq_exchange.h): NCCL grouped
// ncclSend/ncclRecv all-to-allv of partitioned device batches over
// NVLink/NVSwitch, one communicator per GPU/process.  NCCL is dlopen'd
// (libnccl.so.2: the copy torch already loaded, else the system one), so the
// library still loads on machines without it.
#include <algorithm>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/tq_exchange.h"
#include "ctx.h"
#include "device.cuh"
#include "peer.h"

namespace tq {
// exclusive scan of n u32 -> u64 (+ total), ops.cu
void scan_u32_public(tq_ctx* c, const u32* in, u64 n, u64* out, u64* total_dev, cudaStream_t st);
namespace {

struct Nccl {
  bool ok = false;
  ncclResult_t (*get_unique_id)(ncclUniqueId*);
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*destroy)(ncclComm_t);
  ncclResult_t (*group_start)();
  ncclResult_t (*group_end)();
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  const char* (*err)(ncclResult_t);
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("/usr/lib/x86_64-linux-gnu/libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.get_unique_id = (decltype(n.get_unique_id))dlsym(h, "ncclGetUniqueId");
    n.init_rank = (decltype(n.init_rank))dlsym(h, "ncclCommInitRank");
    n.destroy = (decltype(n.destroy))dlsym(h, "ncclCommDestroy");
    n.group_start = (decltype(n.group_start))dlsym(h, "ncclGroupStart");
    n.group_end = (decltype(n.group_end))dlsym(h, "ncclGroupEnd");
    n.send = (decltype(n.send))dlsym(h, "ncclSend");
    n.recv = (decltype(n.recv))dlsym(h, "ncclRecv");
    n.all_gather = (decltype(n.all_gather))dlsym(h, "ncclAllGather");
    n.err = (decltype(n.err))dlsym(h, "ncclGetErrorString");
    n.ok = n.get_unique_id && n.init_rank && n.destroy && n.group_start && n.group_end && n.send && n.recv &&
           n.all_gather && n.err;
  });
  if (!n.ok) fail(TQ_WORKER_FAILURE, "libnccl.so.2 not available");
  return n;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(TQ_PEER_DISCONNECTED, std::string(what) + ": " + nccl().err(r));
}

// bitmap (or all-valid) -> one byte per row
__global__ void k_utf8_lengths(const int32_t* off, u64 n, u32* len) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    len[i] = (u32)(off[i + 1] - off[i]);
}
__global__ void k_u64_to_i32(const u64* in, u64 n, int32_t* out) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    out[i] = (int32_t)in[i];
}

__global__ void k_bits_to_bytes(const uint8_t* bm, u64 n, uint8_t* out) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    out[i] = bm ? ((bm[i >> 3] >> (i & 7)) & 1) : 1;
}
// one byte per row -> LSB-first bitmap (8 rows per thread, whole bytes)
__global__ void k_bytes_to_bits(const uint8_t* in, u64 n, uint8_t* bm) {
  u64 nb = (n + 7) / 8;
  for (u64 b = (u64)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (u64)gridDim.x * blockDim.x) {
    uint8_t v = 0;
    for (int k = 0; k < 8; ++k) {
      u64 i = b * 8 + k;
      if (i < n && in[i]) v |= (uint8_t)(1u << k);
    }
    bm[b] = v;
  }
}

}  // namespace
}  // namespace tq

struct tq_comm {
  tq_ctx* ctx;
  ncclComm_t comm;
  int rank, n;
  std::atomic<uint64_t> sent{0};
  // receive window for the fused partition + NVLink scatter (peer.h): one
  // cudaMalloc'd buffer per rank, mapped into every other rank with CUDA IPC
  uint8_t* win = nullptr;
  uint64_t win_bytes = 0;
  std::vector<uint8_t*> win_peer;  // [n]; win_peer[rank] == win
  uint64_t win_cap_rows = 0;       // most rows any rank received in the last fused exchange (identical on every rank)
  // the window is used as two halves, alternating per fused exchange (epoch parity)
  uint64_t epoch = 0;
};

using namespace tq;

// ---- peer windows (peer.h)
namespace tq {

tq_ctx* comm_ctx(tq_comm* cm) { return cm->ctx; }
int comm_rank(tq_comm* cm) { return cm->rank; }
int comm_size(tq_comm* cm) { return cm->n; }
uint64_t& comm_last_cap(tq_comm* cm) { return cm->win_cap_rows; }
uint64_t& comm_epoch(tq_comm* cm) { return cm->epoch; }
void comm_add_sent(tq_comm* cm, uint64_t bytes) { cm->sent += bytes; }

void comm_allgather_u64(tq_comm* cm, const unsigned long long* dev_in, unsigned long long* dev_out, uint64_t count, cudaStream_t st) {
  nccl_check(nccl().all_gather(dev_in, dev_out, count, ncclUint64, cm->comm, st), "ncclAllGather");
}

void peer_barrier(tq_comm* cm, cudaStream_t st) {
  if (cm->n == 1) return;
  // stream-ordered: work after this point starts only once every rank's prior
  // stream work (their scatter kernels) has completed
  tq_ctx* c = cm->ctx;
  u64* b = (u64*)dalloc(c, 8 * (cm->n + 1), st);
  TQ_CUDA(cudaMemsetAsync(b, 0, 8, st));
  comm_allgather_u64(cm, b, b + 1, 1, st);
  dfree(c, b, 8 * (cm->n + 1), st);
}

uint64_t comm_window_bytes(tq_comm* cm) { return cm->win_bytes; }

PeerView peer_window(tq_comm* cm, uint64_t bytes, cudaStream_t st, bool agreed) {
  tq_ctx* c = cm->ctx;
  const int n = cm->n;
  if (!agreed) {
    // every rank must see the same size: take the max over ranks
    u64* g = (u64*)dalloc(c, 8 * (n + 1), st);
    TQ_CUDA(cudaMemcpyAsync(g, &bytes, 8, cudaMemcpyHostToDevice, st));
    comm_allgather_u64(cm, g, g + 1, 1, st);
    std::vector<u64> all(n);
    TQ_CUDA(cudaMemcpyAsync(all.data(), g + 1, 8 * n, cudaMemcpyDeviceToHost, st));
    TQ_CUDA(cudaStreamSynchronize(st));
    dfree(c, g, 8 * (n + 1), st);
    for (u64 v : all) bytes = std::max<u64>(bytes, v);
  }
  // (agreed: every rank passes the same `bytes`, so every rank takes the same
  // grow / no-grow branch and the collectives below stay matched)
  if (cm->win_bytes < bytes) {
    // drop the old mappings and buffer (every peer finished with them: the
    // previous scatter ended with a barrier and its copy-out is stream-ordered)
    TQ_CUDA(cudaStreamSynchronize(st));
    peer_barrier(cm, st);
    TQ_CUDA(cudaStreamSynchronize(st));
    for (int p = 0; p < (int)cm->win_peer.size(); ++p)
      if (p != cm->rank && cm->win_peer[p]) cudaIpcCloseMemHandle(cm->win_peer[p]);
    if (cm->win) cudaFree(cm->win);
    cm->win = nullptr;
    cm->win_peer.assign(n, nullptr);
    const u64 alloc = round_up(std::max<u64>(bytes, 1ull << 20) * 5 / 4, 1ull << 21);
    TQ_CUDA(cudaMalloc(&cm->win, alloc));  // plain cudaMalloc: exportable with cudaIpcGetMemHandle
    cm->win_bytes = alloc;
    cudaIpcMemHandle_t h;
    TQ_CUDA(cudaIpcGetMemHandle(&h, cm->win));
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
    u64* hd = (u64*)dalloc(c, 64 * (n + 1), st);
    TQ_CUDA(cudaMemcpyAsync(hd, &h, 64, cudaMemcpyHostToDevice, st));
    comm_allgather_u64(cm, hd, hd + 8, 8, st);
    std::vector<cudaIpcMemHandle_t> hs(n);
    TQ_CUDA(cudaMemcpyAsync(hs.data(), hd + 8, 64 * n, cudaMemcpyDeviceToHost, st));
    TQ_CUDA(cudaStreamSynchronize(st));
    dfree(c, hd, 64 * (n + 1), st);
    for (int p = 0; p < n; ++p) {
      if (p == cm->rank) {
        cm->win_peer[p] = cm->win;
        continue;
      }
      void* ptr = nullptr;
      TQ_CUDA(cudaIpcOpenMemHandle(&ptr, hs[p], cudaIpcMemLazyEnablePeerAccess));
      cm->win_peer[p] = (uint8_t*)ptr;
    }
  }
  PeerView v;
  v.local = cm->win;
  v.peer = cm->win_peer;
  v.rank = cm->rank;
  v.n = n;
  return v;
}

}  // namespace tq

namespace {

// Core all-to-allv.  send_off/send_cnt: rows of `in` for each peer (host).
void exchange_impl(tq_comm* cm, const tq_batch* in, const std::vector<uint64_t>& send_off,
                   const std::vector<uint64_t>& send_cnt, tq_batch* out, uint64_t* recv_offsets, cudaStream_t st) {
  tq_ctx* c = cm->ctx;
  Nccl& N = nccl();
  const int n = cm->n, me = cm->rank;
  if (in->mem != TQ_MEM_DEVICE) fail(TQ_INTERNAL, "exchange needs a device batch");
  if (in->ncols > 62) fail(TQ_INVALID_PLAN, "too many columns to exchange");
  // Utf8 columns travel as per-row lengths (int32) + the bytes of each part's
  // row range; the receiver rebuilds the offsets by a scan over the lengths
  std::vector<uint32_t> ucols;
  for (uint32_t k = 0; k < in->ncols; ++k)
    if (in->cols[k].kind == TQ_UTF8) ucols.push_back(k);
  const int nu = (int)ucols.size();
  // per Utf8 column and peer: the byte range [ustart, uend) of the rows sent to it
  // (parts of a partition are adjacent; an all-gather sends every peer all rows)
  std::vector<std::vector<int32_t>> ustart(nu, std::vector<int32_t>(n, 0)), uend(nu, std::vector<int32_t>(n, 0));
  std::vector<u32*> ulen(nu, nullptr);
  const u64 in_len_bytes = std::max<u64>(4, in->rows * 4);
  if (nu) {
    if ((u64)2 * n * nu * 4 > 4096) fail(TQ_INVALID_PLAN, "too many utf8 columns for one exchange");
    int32_t* pin = (int32_t*)pinned_scratch(c);  // 2 n nu ints <= 4 KB
    for (int j = 0; j < nu; ++j) {
      const tq_column& col = in->cols[ucols[j]];
      for (int p = 0; p < n; ++p) {
        TQ_CUDA(cudaMemcpyAsync(pin + (j * n + p) * 2, col.offsets + send_off[p], 4, cudaMemcpyDeviceToHost, st));
        TQ_CUDA(cudaMemcpyAsync(pin + (j * n + p) * 2 + 1, col.offsets + send_off[p] + send_cnt[p], 4,
                                cudaMemcpyDeviceToHost, st));
      }
      ulen[j] = (u32*)dalloc(c, in_len_bytes, st);
      if (in->rows)
        k_utf8_lengths<<<(u32)std::max<u64>(1, std::min<u64>((in->rows + 255) / 256, 4096)), 256, 0, st>>>(
            col.offsets, in->rows, ulen[j]);
      counted_launch(c);
    }
    TQ_CUDA(cudaStreamSynchronize(st));
    for (int j = 0; j < nu; ++j)
      for (int p = 0; p < n; ++p) {
        ustart[j][p] = pin[(j * n + p) * 2];
        uend[j][p] = pin[(j * n + p) * 2 + 1];
      }
  }
  // 1) header all-gather: counts for every peer + a validity-presence mask
  //    (+ per Utf8 column, the bytes for every peer)
  const int hw = n + 1 + n * nu;
  u64* hdr = (u64*)dalloc(c, (size_t)hw * (n + 1) * 8, st);
  std::vector<u64> mine(hw);
  for (int p = 0; p < n; ++p) mine[p] = send_cnt[p];
  u64 vmask = 0;
  for (uint32_t k = 0; k < in->ncols; ++k)
    if (in->rows > 0 && in->cols[k].validity) vmask |= 1ull << k;
  mine[n] = vmask;
  for (int j = 0; j < nu; ++j)
    for (int p = 0; p < n; ++p) mine[n + 1 + j * n + p] = (u64)(uend[j][p] - ustart[j][p]);
  TQ_CUDA(cudaMemcpyAsync(hdr + (size_t)hw * n, mine.data(), hw * 8, cudaMemcpyHostToDevice, st));
  nccl_check(N.all_gather(hdr + (size_t)hw * n, hdr, hw, ncclUint64, cm->comm, st), "ncclAllGather");
  std::vector<u64> all((size_t)hw * n);
  TQ_CUDA(cudaMemcpyAsync(all.data(), hdr, all.size() * 8, cudaMemcpyDeviceToHost, st));
  TQ_CUDA(cudaStreamSynchronize(st));
  dfree(c, hdr, (size_t)hw * (n + 1) * 8, st);
  std::vector<uint64_t> recv_cnt(n), recv_off(n + 1, 0);
  u64 any_valid = 0;
  for (int s = 0; s < n; ++s) {
    recv_cnt[s] = all[(size_t)s * hw + me];
    recv_off[s + 1] = recv_off[s] + recv_cnt[s];
    any_valid |= all[(size_t)s * hw + n];
  }
  if (recv_offsets)
    for (int s = 0; s <= n; ++s) recv_offsets[s] = recv_off[s];
  const uint64_t rows = recv_off[n];
  // Utf8: received bytes per source (in source order) and in total
  std::vector<std::vector<u64>> ubyte_off(nu, std::vector<u64>(n + 1, 0));
  std::vector<uint64_t> ub(in->ncols, 0);
  for (int j = 0; j < nu; ++j) {
    for (int s = 0; s < n; ++s) ubyte_off[j][s + 1] = ubyte_off[j][s] + all[(size_t)s * hw + n + 1 + j * n + me];
    if (ubyte_off[j][n] > 0x7fffffffull) fail(TQ_INVALID_PLAN, "utf8 column over 2 GiB after the exchange");
    ub[ucols[j]] = ubyte_off[j][n];
  }
  // 2) output batch
  std::vector<tq_column> sch(in->cols, in->cols + in->ncols);
  std::vector<bool> wv;
  for (uint32_t k = 0; k < in->ncols; ++k) wv.push_back((any_valid >> k) & 1);
  alloc_batch(c, rows, sch, wv, out, st, &ub);
  const u64 out_len_bytes = std::max<u64>(4, rows * 4);
  std::vector<u32*> urecv(nu, nullptr);
  for (int j = 0; j < nu; ++j) urecv[j] = (u32*)dalloc(c, out_len_bytes, st);
  // validity travels as one byte per row
  uint8_t* vsend = nullptr;
  uint8_t* vrecv = nullptr;
  const int nv = __builtin_popcountll(any_valid);
  if (nv) {
    vsend = (uint8_t*)dalloc(c, std::max<u64>(1, in->rows) * nv, st);
    vrecv = (uint8_t*)dalloc(c, std::max<u64>(1, rows) * nv, st);
    int j = 0;
    for (uint32_t k = 0; k < in->ncols; ++k) {
      if (!((any_valid >> k) & 1)) continue;
      if (in->rows)
        k_bits_to_bytes<<<std::max<u64>(1, std::min<u64>((in->rows + 255) / 256, 4096)), 256, 0, st>>>(
            in->rows ? in->cols[k].validity : nullptr, in->rows, vsend + (u64)j * in->rows);
      counted_launch(c);
      ++j;
    }
  }
  // 3) grouped point-to-point transfers, one per (peer, column)
  u64 sent = 0;
  nccl_check(N.group_start(), "ncclGroupStart");
  for (int p = 0; p < n; ++p) {
    int j = 0;
    for (uint32_t k = 0; k < in->ncols; ++k) {
      if (in->cols[k].kind == TQ_UTF8) {
        const int j = (int)(std::find(ucols.begin(), ucols.end(), k) - ucols.begin());
        const u64 sb = (u64)(uend[j][p] - ustart[j][p]);
        const u64 rb = ubyte_off[j][p + 1] - ubyte_off[j][p];
        if (send_cnt[p]) {
          nccl_check(N.send(ulen[j] + send_off[p], send_cnt[p] * 4, ncclUint8, p, cm->comm, st), "ncclSend");
          if (sb)
            nccl_check(N.send((const uint8_t*)in->cols[k].values + ustart[j][p], sb, ncclUint8, p, cm->comm, st),
                       "ncclSend");
        }
        if (recv_cnt[p]) {
          nccl_check(N.recv(urecv[j] + recv_off[p], recv_cnt[p] * 4, ncclUint8, p, cm->comm, st), "ncclRecv");
          if (rb)
            nccl_check(N.recv((uint8_t*)out->cols[k].values + ubyte_off[j][p], rb, ncclUint8, p, cm->comm, st),
                       "ncclRecv");
        }
        if (p != me) sent += send_cnt[p] * 4 + sb;
      } else {
        const size_t w = width_of(in->cols[k].kind);
        const uint8_t* sv = (const uint8_t*)in->cols[k].values;
        uint8_t* rv = (uint8_t*)out->cols[k].values;
        if (send_cnt[p]) nccl_check(N.send(sv + send_off[p] * w, send_cnt[p] * w, ncclUint8, p, cm->comm, st), "ncclSend");
        if (recv_cnt[p]) nccl_check(N.recv(rv + recv_off[p] * w, recv_cnt[p] * w, ncclUint8, p, cm->comm, st), "ncclRecv");
        if (p != me) sent += send_cnt[p] * w;
      }
      if ((any_valid >> k) & 1) {
        if (send_cnt[p])
          nccl_check(N.send(vsend + (u64)j * in->rows + send_off[p], send_cnt[p], ncclUint8, p, cm->comm, st), "ncclSend");
        if (recv_cnt[p])
          nccl_check(N.recv(vrecv + (u64)j * rows + recv_off[p], recv_cnt[p], ncclUint8, p, cm->comm, st), "ncclRecv");
        if (p != me) sent += send_cnt[p];
        ++j;
      }
    }
  }
  nccl_check(N.group_end(), "ncclGroupEnd");
  cm->sent += sent;
  if (nv) {
    int j = 0;
    for (uint32_t k = 0; k < in->ncols; ++k) {
      if (!((any_valid >> k) & 1)) continue;
      if (rows)
        k_bytes_to_bits<<<std::max<u64>(1, std::min<u64>((rows / 8 + 255) / 256, 4096)), 256, 0, st>>>(
            vrecv + (u64)j * rows, rows, out->cols[k].validity);
      counted_launch(c);
      ++j;
    }
    dfree(c, vsend, std::max<u64>(1, in->rows) * nv, st);
    dfree(c, vrecv, std::max<u64>(1, rows) * nv, st);
  }
  // Utf8 offsets of the output: exclusive scan of the received lengths
  for (int j = 0; j < nu; ++j) {
    u64* scan = (u64*)dalloc(c, (rows + 1) * 8, st);
    scan_u32_public(c, urecv[j], rows, scan, scan + rows, st);
    k_u64_to_i32<<<(u32)std::max<u64>(1, std::min<u64>((rows + 1 + 255) / 256, 4096)), 256, 0, st>>>(
        scan, rows + 1, out->cols[ucols[j]].offsets);
    counted_launch(c);
    dfree(c, scan, (rows + 1) * 8, st);
    dfree(c, urecv[j], out_len_bytes, st);
    dfree(c, ulen[j], in_len_bytes, st);
  }
  TQ_CUDA(cudaGetLastError());
}

}  // namespace

extern "C" {

tq_status tq_comm_unique_id(uint8_t* id) {
  return guard([&] {
    ncclUniqueId u;
    nccl_check(nccl().get_unique_id(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
  });
}

tq_status tq_comm_init(tq_ctx* c, int rank, int nranks, const uint8_t* id, tq_comm** out) {
  return guard([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(TQ_INVALID_PLAN, "bad rank");
    TQ_CUDA(cudaSetDevice(c->device));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    ncclComm_t comm;
    nccl_check(nccl().init_rank(&comm, nranks, u, rank), "ncclCommInitRank");
    tq_comm* cm = new tq_comm();
    cm->ctx = c;
    cm->comm = comm;
    cm->rank = rank;
    cm->n = nranks;
    *out = cm;
  });
}

void tq_comm_destroy(tq_comm* cm) {
  if (!cm) return;
  for (int p = 0; p < (int)cm->win_peer.size(); ++p)
    if (p != cm->rank && cm->win_peer[p]) cudaIpcCloseMemHandle(cm->win_peer[p]);
  if (cm->win) cudaFree(cm->win);
  try {
    nccl().destroy(cm->comm);
  } catch (...) {
  }
  delete cm;
}

tq_status tq_comm_exchange(tq_comm* cm, const tq_batch* in, const uint64_t* part_offsets, tq_batch* out,
                           uint64_t* recv_offsets, void* stream) {
  return guard([&] {
    std::vector<uint64_t> off(cm->n), cnt(cm->n);
    for (int p = 0; p < cm->n; ++p) {
      off[p] = part_offsets[p];
      cnt[p] = part_offsets[p + 1] - part_offsets[p];
    }
    if (part_offsets[cm->n] != in->rows) fail(TQ_INVALID_PLAN, "part offsets do not cover the batch");
    exchange_impl(cm, in, off, cnt, out, recv_offsets, pick(cm->ctx, stream));
  });
}

tq_status tq_comm_allgather(tq_comm* cm, const tq_batch* in, tq_batch* out, uint64_t* recv_offsets, void* stream) {
  return guard([&] {
    std::vector<uint64_t> off(cm->n, 0), cnt(cm->n, in->rows);
    cudaStream_t st = pick(cm->ctx, stream);
    const int ph = prof_begin(cm->ctx, "nccl_allgather", st);
    exchange_impl(cm, in, off, cnt, out, recv_offsets, st);
    prof_end(cm->ctx, ph, st);
  });
}

uint64_t tq_comm_bytes_sent(tq_comm* cm) { return cm->sent.load(); }

tq_status tq_comm_bloom_union(tq_comm* cm, tq_bloom* b, void* stream) {
  return guard([&] {
    if (cm->n == 1) return;
    tq_ctx* c = cm->ctx;
    cudaStream_t st = pick(c, stream);
    const uint64_t nw = tq_bloom_words(b);
    uint32_t* all = (uint32_t*)dalloc(c, nw * 4 * cm->n, st);
    nccl_check(nccl().all_gather(tq_bloom_data(b), all, nw, ncclUint32, cm->comm, st), "ncclAllGather");
    cm->sent += nw * 4 * (cm->n - 1);
    tq_status r = tq_bloom_or_gathered(b, all, cm->n, st);
    dfree(c, all, nw * 4 * cm->n, st);
    if (r != TQ_OK) fail(r, g_err);
  });
}
int tq_comm_size(tq_comm* cm) { return cm->n; }
int tq_comm_rank(tq_comm* cm) { return cm->rank; }

}  // extern "C"

// ---- AdaptiveExchange control
extern "C" {

tq_status tq_comm_allgather_host_u64(tq_comm* cm, const uint64_t* in, uint64_t* out, uint64_t count, void* stream) {
  return guard([&] {
    tq_ctx* c = cm->ctx;
    cudaStream_t st = pick(c, stream);
    const uint64_t n = (uint64_t)cm->n;
    u64* g = (u64*)dalloc(c, 8 * count * (n + 1), st);
    // staged through this thread's pinned slot: asynchronous copies, one sync
    u64* pin = (u64*)pinned_scratch(c);
    const bool fits = 8 * count * (n + 1) <= 4096;
    if (fits) std::memcpy(pin, in, 8 * count);
    TQ_CUDA(cudaMemcpyAsync(g, fits ? (const void*)pin : (const void*)in, 8 * count, cudaMemcpyHostToDevice, st));
    comm_allgather_u64(cm, g, g + count, count, st);
    TQ_CUDA(cudaMemcpyAsync(fits ? (void*)(pin + count) : (void*)out, g + count, 8 * count * n, cudaMemcpyDeviceToHost,
                            st));
    TQ_CUDA(cudaStreamSynchronize(st));
    if (fits) std::memcpy(out, pin + count, 8 * count * n);
    dfree(c, g, 8 * count * (n + 1), st);
  });
}

int tq_exchange_phase1(uint64_t bytes_so_far, double progress, double sample_fraction, uint64_t* estimate) {
  if (progress >= 1.0) {  // scan complete: the bytes are exact (0 for an empty input)
    if (estimate) *estimate = bytes_so_far;
    return 1;
  }
  if (progress <= 0.0 || progress < sample_fraction) return 0;
  if (estimate) *estimate = (uint64_t)((double)bytes_so_far / progress);  // 10 MiB at 25% -> 40 MiB
  return 1;
}

int tq_exchange_decide(const uint64_t* est0, const uint64_t* est1, int n, uint64_t threshold, int* broadcast_side,
                       uint64_t* total0, uint64_t* total1) {
  uint64_t t0 = 0, t1 = 0;
  for (int i = 0; i < n; ++i) {
    t0 += est0[i];
    t1 += est1[i];
  }
  if (total0) *total0 = t0;
  if (total1) *total1 = t1;
  if (std::min(t0, t1) <= threshold * (uint64_t)n) {
    if (broadcast_side) *broadcast_side = t0 <= t1 ? 0 : 1;
    return TQ_XCHG_BROADCAST;
  }
  if (broadcast_side) *broadcast_side = -1;
  return TQ_XCHG_HASH_PARTITION;
}

}  // extern "C"
