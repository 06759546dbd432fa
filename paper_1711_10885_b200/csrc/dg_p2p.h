#pragma once
// Direct (fused) face-trace halo: the trace pack kernel stores every partition face's traces
// straight into the neighbour rank's receive buffer -- over NVLink through a CUDA IPC mapping of the
// peer's buffer (ranks as processes, one per GPU), or through the plain pointer when the ranks are
// threads of one process -- so the compute step and the transfer are one kernel and there is no
// separate collective (SURVEY 8(e) "fused collective"; the NCCL path sends from a send buffer).
//
// Per apply t of rank r (every rank applies collectively):
//   before_pack  : the comm stream waits until every neighbour has finished reading what r
//                  wrote into it in apply t-1 (the neighbour's "consumed" event of t-1);
//   pack         : trace_pack_kernel with the neighbours' receive buffers as destinations;
//   after_pack   : r records its "packed" event and posts t;
//   before_shell : the compute stream waits for every neighbour's "packed" event of t;
//   shell kernel : reads the receive buffers;
//   after_shell  : r records its "consumed" event and posts t.
// A host-side counter per rank and event (in the process for threads, in a POSIX shared-memory
// segment for processes) orders each record before the peers' waits on it: no kernel ever spins
// on another rank, every cross-rank dependency is a stream wait on an event already recorded.
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace dg {

struct P2P;

// in-process (ranks as threads): join the group `key` as `rank` of `nranks` with this rank's
// receive buffers recv[6]; peers are resolved at the first exchange. 0 ok, -1 error.
int p2p_local_join(uint64_t key, int rank, int nranks, const int nbr[6], double* const recv[6], P2P** out);
// multi-process: this rank's export blob (IPC handles of recv[6] and of its two events)
size_t p2p_blob_bytes();
int p2p_ipc_create(int rank, int nranks, const int nbr[6], double* const recv[6], P2P** out);
int p2p_ipc_export(const P2P* p, void* blob);
// open the neighbours' buffers and events from all ranks' blobs (nranks x p2p_blob_bytes()) and the
// shared-memory segment `shm_name` (rank 0 creates it). 0 ok, -1 error.
int p2p_ipc_import(P2P* p, const void* blobs, const char* shm_name);
void p2p_destroy(P2P* p);

// where this rank's face-f traces go (the neighbour's receive buffer of face f^1), nullptr: none
double* p2p_remote(const P2P* p, int face);
// the per-apply protocol above; 0 ok, -1 timeout / error, -2 CUDA error
int p2p_before_pack(P2P* p, cudaStream_t comm);
int p2p_after_pack(P2P* p, cudaStream_t comm);
int p2p_before_shell(P2P* p, cudaStream_t s);
int p2p_after_shell(P2P* p, cudaStream_t s);
bool p2p_ready(const P2P* p);   // the peers are resolved (import done / all threads joined)

}  // namespace dg
