// peer.h — receive windows shared over NVLink with CUDA IPC (exchange.cu),
// used by the fused partition + scatter (ops.cu, tq_pipeline_partition_exchange).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/tq_exchange.h"

namespace tq {

// Window layout (identical on every rank): two halves of win_bytes / 2, used
// alternately by successive fused exchanges; each half: [0, 256) control word
// = the row counter; [256, 256 + n * kMaxTailCtas * 16) tail slots {base, used}
// per (source rank, CTA); then the data region (column values / bitmaps).
struct PeerView {
  uint8_t* local = nullptr;     // this rank's window
  std::vector<uint8_t*> peer;   // [n] every rank's window as mapped in this process
  int rank = 0, n = 1;
};

// Collective: every rank calls with its wanted size; all get a window of at
// least the max over ranks (re-allocated and re-mapped only when it grows).
// agreed = every rank passes the same size: no size all-gather, no host sync.
PeerView peer_window(tq_comm* cm, uint64_t bytes, cudaStream_t st, bool agreed = false);
// Current window size (identical on every rank: windows only grow collectively).
uint64_t comm_window_bytes(tq_comm* cm);
// Collective stream-ordered barrier (a one-word NCCL all-gather).
void peer_barrier(tq_comm* cm, cudaStream_t st);
void comm_allgather_u64(tq_comm* cm, const unsigned long long* dev_in, unsigned long long* dev_out, uint64_t count, cudaStream_t st);
tq_ctx* comm_ctx(tq_comm* cm);
int comm_rank(tq_comm* cm);
int comm_size(tq_comm* cm);
uint64_t& comm_epoch(tq_comm* cm);                // fused exchanges completed (same on every rank)
uint64_t& comm_last_cap(tq_comm* cm);  // rows capacity of the last fused exchange (same on every rank)
void comm_add_sent(tq_comm* cm, uint64_t bytes);  // NVLink bytes accounting

}  // namespace tq
