// Private multi-GPU halo layer of libfastilu_b200.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/fastilu.h"
#include "device.h"

namespace fastilu {

struct Comm;

// Collective over the ranks of opts: exchanges the partition (row_begin, n, G, H) of every rank
// and validates that ghost rows come only from the immediate neighbours.
// Also sums `stat` (e.g. the number of strict-lower entries) over ranks into *stat_global so
// that launch shapes that affect rounding (the trisolve's lanes per row) are chosen from global
// statistics and results stay bitwise independent of the partition.
fastilu_status comm_setup(Comm *&out, const fastilu_options &opts, int64_t row_begin, int64_t n,
                          int64_t G, int64_t H, const int64_t *h_rp_local, int64_t stat,
                          int64_t *stat_global, int tsell_W, uint64_t layout_hash,
                          cudaStream_t st);
// Vector halo on an extended vector [G | n | H]: lower ghosts from rank-1's last G owned
// entries, upper ghosts from rank+1's first H owned entries.
fastilu_status comm_vector_halo(Comm *c, double *x, cudaStream_t st, bool lower, bool upper);
// Factor halo before a sweep: the G ghost rows' values (whole rows: CSR S order, or whole
// 32-row template slices when tsell_W > 0) and their
// diagonal copies from rank-1.
fastilu_status comm_factor_halo(Comm *c, double *vals, const int64_t *d_rp, double *udiag,
                                cudaStream_t st);
// Host-side sum of the residual history and min of the (GLOBAL-index) error flags over ranks.
fastilu_status comm_allreduce_host(Comm *c, double *r2, int count, ErrFlags &ef);
void comm_destroy(Comm *c);

}  // namespace fastilu
