// Row-wise assembly helpers shared by the tet builders (host_tet.cpp,
// host_p2.cpp).
#pragma once
#include <algorithm>
#include <utility>
#include <vector>

#include "common.hpp"

namespace sfeec_b200 {

// Generic per-row assembly: row r gathers the local contributions of its
// containing tets in ascending tet id, sums from 0.0, drops exact zeros.
template <class RowFn>
inline HostCSR assemble_rows(int64_t rows, int64_t cols, int max_row, RowFn&& fn) {
  HostCSR m;
  m.rows = rows;
  m.cols = cols;
  m.row_ptr.assign((size_t)rows + 1, 0);
  std::vector<int32_t> tc((size_t)rows * max_row);
  std::vector<double> tv((size_t)rows * max_row);
  std::vector<int32_t> cnt((size_t)rows);
  bool overflow = false;
#pragma omp parallel
  {
    std::vector<std::pair<int32_t, double>> acc;
#pragma omp for schedule(dynamic, 1024)
    for (int64_t r = 0; r < rows; ++r) {
      acc.clear();
      fn(r, acc);
      std::sort(acc.begin(), acc.end(),
                [](const auto& a, const auto& b) { return a.first < b.first; });
      int w = 0;
      for (auto& pr : acc)
        if (pr.second != 0.0) {
          if (w < max_row) {
            tc[(size_t)r * max_row + w] = pr.first;
            tv[(size_t)r * max_row + w] = pr.second;
          }
          ++w;
        }
      if (w > max_row) overflow = true;
      cnt[(size_t)r] = w;
    }
  }
  require(!overflow, "assembly: row longer than expected");
  for (int64_t r = 0; r < rows; ++r) m.row_ptr[(size_t)r + 1] = m.row_ptr[(size_t)r] + cnt[(size_t)r];
  m.col_idx.resize((size_t)m.row_ptr[(size_t)rows]);
  m.val.resize((size_t)m.row_ptr[(size_t)rows]);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r)
    for (int k = 0; k < cnt[(size_t)r]; ++k) {
      m.col_idx[(size_t)(m.row_ptr[(size_t)r] + k)] = tc[(size_t)r * max_row + k];
      m.val[(size_t)(m.row_ptr[(size_t)r] + k)] = tv[(size_t)r * max_row + k];
    }
  return m;
}

// accumulate v into the (col -> sum) list, first occurrence keeps order of
// arrival; duplicates are summed in arrival order (ascending tets)
inline void add_to(std::vector<std::pair<int32_t, double>>& acc, int32_t c, double v) {
  for (auto& p : acc)
    if (p.first == c) {
      p.second = p.second + v;
      return;
    }
  acc.push_back({c, 0.0 + v});
}

}  // namespace sfeec_b200
