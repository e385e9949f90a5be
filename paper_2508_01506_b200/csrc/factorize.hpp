// factorize.hpp -- batched device rank-r factorization.
//
// Replaces factor_rank_r (svd.cpp:412-456) for a whole batch of matrices at
// once: every block of every layer of a model is factorized in one device
// run instead of one serial CPU Jacobi per matrix.
#pragma once

#include <cstddef>
#include <vector>

namespace fsvd {

// One rank-r factorization: a is a host row-major m x n matrix with leading
// dimension lda (>= n); u (m x r) and v (r x n) are host row-major outputs.
struct FactorJob {
  const float* a;
  size_t lda, m, n, r;
  float* u;
  float* v;
};

// Validates every job the way factor_rank_r does (RankError), then factorizes
// the whole batch on the current device.  Outputs follow the reference
// contract: A ~ U V with the even singular-value split, leading-r singular
// triplets in descending order, the largest-magnitude entry of each U column
// positive, zero factors for singular values <= 1e-15 * sigma_max.
void factor_rank_r_batch(const std::vector<FactorJob>& jobs);

// factor_rank_r's argument checks alone (host, no device needed).
void check_factor_job(size_t m, size_t n, size_t r);

// Jacobi sweeps the last batch needed (max over its jobs); for tests / bench.
int last_factor_sweeps();

}  // namespace fsvd
