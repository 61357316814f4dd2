// Device generation of the reference's initial random blocks.
#pragma once

#include "common.hpp"

namespace bosp {
inline namespace b200 {

// Fill U (n x d) then V (n x d), column by column, with the mt19937_64(seed) +
// uniform_real_distribution(-1, 1) stream -- bit-identical to the reference's
// x,p,w,y,q,z fill order when U = [X | P | W] and V = [Y | Q | Z] (bosp_solver.cpp:144-150).
// Row-partitioned: the stream is drawn over n_global rows and this rank keeps rows
// [row0, row0 + u.rows) (n_global <= 0 -> unpartitioned).
void mt_fill_uv(uint64_t seed, const DMat& u, const DMat& v, int64_t n_global = 0, int64_t row0 = 0);

}  // namespace b200
}  // namespace bosp
