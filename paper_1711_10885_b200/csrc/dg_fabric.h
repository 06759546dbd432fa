#pragma once
// In-process halo fabric: the ranks of one partitioned operator as threads of ONE process
// (contexts on one or several devices), exchanging the halo with stream-ordered copies and
// cross-stream events instead of NCCL. It implements NCCL's point-to-point semantics the
// transport relies on (per ordered rank pair, the i-th send matches the i-th receive), so the
// orchestration of dg_apply on a partitioned box -- trace pack on the comm stream, the
// exchange, the inner-box kernel overlapping it, the shell kernel after the receive event --
// runs unchanged on a single GPU. No kernel ever waits on another rank's
// kernel: every cross-rank dependency is a CUDA event recorded before it is waited on
// (the host rendezvous below guarantees the order), so the DAG is acyclic.
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace dg {

struct Fabric;

bool fabric_id_is(const void* id128);     // an id made by fabric_make_id (not an ncclUniqueId)
void fabric_make_id(void* out128);
// join the group named by id as `rank` of `nranks`; 0 ok, -1 mismatch / resources
int fabric_join(const void* id128, int rank, int nranks, Fabric** out);
void fabric_leave(Fabric* f, int rank);
// Before this rank overwrites its send buffers: stream s waits until every neighbour that
// read them in the previous exchange has finished copying. 0 ok, -1 timeout.
int fabric_prepare(Fabric* f, int rank, const int nbr[6], cudaStream_t s);
// One exchange round, enqueued on s after the send buffers' producer: send[f] (cnt[f] doubles)
// goes to rank nbr[f]; recv[f] receives from nbr[f]; sends issued for faces f = 0..5 and the
// receive of face f^1 after the send of face f (the NCCL group's order). 0 ok, -1 mismatch /
// timeout, -2 CUDA error.
int fabric_exchange(Fabric* f, int rank, const int nbr[6], double* const send[6], double* const recv[6],
                    const size_t cnt[6], cudaStream_t s);

}  // namespace dg
