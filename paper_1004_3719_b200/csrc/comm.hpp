// Communicator layer of the distributed sequence (comm.cpp); internal.
#pragma once

#include <cstddef>
#include <string>

#include "../../include/ffspmv.h"

namespace ffspmv {

struct CommImpl;

// records a thread-local message for ffspmv_last_error() and returns s (abi.cpp)
ffspmv_status set_error(ffspmv_status s, const std::string &msg);

CommImpl *comm_impl(ffspmv_comm c);
int comm_size(const CommImpl *c);
int comm_rank(const CommImpl *c);
// all-gather of `bytes` per rank from send into recv (P chunks); in place
// when send == recv + rank * bytes.  Returns 0, a cudaError_t, or -1 (NCCL).
int comm_allgather(CommImpl *c, const void *send, void *recv, size_t bytes, void *stream,
                   std::string &err);
// collective over c: the ranks with equal color form a new communicator of
// `nranks` ranks, this one being `rank` (ordered by key)
CommImpl *comm_split(CommImpl *c, int color, int key, int nranks, int rank, std::string &err);
void comm_free(CommImpl *c);

}  // namespace ffspmv
