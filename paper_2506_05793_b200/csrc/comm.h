// Private multi-GPU halo layer of libfastilu_b200.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <vector>

#include "../../include/fastilu.h"
#include "device.h"

namespace fastilu {

struct Comm;

// Collective: binds the rank to its transport (NCCL communicator or in-process group).
fastilu_status comm_init(Comm *&out, const fastilu_options &opts, cudaStream_t st);
// Collective all-gather of mine.size() int64 per rank into all[nranks][mine.size()].
fastilu_status comm_allgather_i64(Comm *c, const std::vector<int64_t> &mine,
                                  std::vector<int64_t> &all, cudaStream_t st);
// Collective: exchanges the partition (row_begin, n, G, H) of every rank, validates that ghost
// rows come only from the immediate neighbours and that the ghost/halo sizes match.  Also sums
// `stat` (e.g. the number of strict-lower entries) over ranks into *stat_global so that launch
// shapes that affect rounding are chosen from global statistics (results stay bitwise
// independent of the partition).  tsell_W > 0: template-SELL layout of width W.
fastilu_status comm_layout(Comm *c, int64_t row_begin, int64_t n, int64_t G, int64_t H,
                           const int64_t *h_rp_local, int64_t stat, int64_t *stat_global,
                           int tsell_W, uint64_t layout_hash, cudaStream_t st);
// Vector halo on an extended vector [G | n | H]: lower ghosts from rank-1's last G owned
// entries, upper ghosts from rank+1's first H owned entries.
fastilu_status comm_vector_halo(Comm *c, double *x, cudaStream_t st, bool lower, bool upper);
// The same on the comm's halo stream, after `st`'s work so far; *done marks the ghosts in place
// (the caller overlaps the rows that read no ghost entry).
fastilu_status comm_vector_halo_async(Comm *c, double *x, cudaStream_t st, bool lower,
                                      bool upper, cudaEvent_t *done);
// Factor halo before a sweep: the G ghost rows' values (whole rows: CSR S order, or whole
// 32-row template slices when tsell_W > 0) and their
// diagonal copies from rank-1.
fastilu_status comm_factor_halo(Comm *c, double *vals, const int64_t *d_rp, double *udiag,
                                cudaStream_t st);
// Template layout: the factor halo of a sweep restricted to what the sweep kernels read from a
// ghost row -- columns [c0, W) (diagonal + strict upper part) -- packed into one contiguous
// message per neighbour (about half of whole rows), on the comm's own halo stream after the
// iterate is complete on `st`; unpacked into the ghost slices (+ udiag).  *done is recorded on
// the halo stream when the ghost rows are in place: the caller sweeps the rows that read no
// ghost row meanwhile and waits on *done before the others.
fastilu_status comm_factor_halo_upper(Comm *c, double *vals, double *udiag, int W, int c0,
                                      cudaStream_t st, cudaEvent_t *done);
// bytes this rank sends per factor halo (template: packed columns; CSR: whole rows)
int64_t comm_halo_bytes(const Comm *c, int W, int c0);
// Host-side sum of the residual history and min of the (GLOBAL-index) error flags over ranks.
fastilu_status comm_allreduce_host(Comm *c, double *r2, int count, ErrFlags &ef);
void comm_destroy(Comm *c);

}  // namespace fastilu
