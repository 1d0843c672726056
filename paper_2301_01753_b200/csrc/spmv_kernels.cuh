// Device sparse operators and the SpMV kernels of the leapfrog chain
// (K-Q, K-Cb, K-M2, K-CTe in SURVEY.md 2.4).
#pragma once
#include <memory>
#include <vector>

#include "device_util.cuh"

namespace sfeec_b200 {

// Device copy of one operator. The CSR arrays are always kept (strict mode,
// export); production mode adds a sliced layout when it pays:
//   slices: runs of <= 32 consecutive rows of (nearly) equal length, chosen
//           greedily from the row lengths (the tet numbering groups rows of
//           one entity type, so slices are full and unpadded). Inside a slice
//           entry k of row r sits at slice_ptr + k*rows_in_slice + (r - first
//           row): one warp streams a slice with contiguous loads, one lane
//           per row, no shuffles, rows summed in CSR order.
//   kSigned: every |value| equals one scalar (incidence matrices: +-1 for the
//            Whitney P1- curl); one int32 per entry, sign in the top bit
//            (~col for negative) -> 4 B/entry instead of 12.
//   kSell:   general values: fp64 value + int32 column per entry.
struct DevOperator {
  enum Layout { kCsr = 0, kSigned = 1, kSell = 2 };
  int64_t rows = 0, cols = 0, nnz = 0;
  DevBuf<int64_t> rp;
  DevBuf<int32_t> ci;
  DevBuf<double> val;
  int tpr = 1;  // threads per row for the CSR-vector kernel
  Layout layout = kCsr;
  int64_t n_slices = 0, sell_entries = 0;
  DevBuf<int64_t> slice_row;  // first row of each slice (n_slices + 1)
  DevBuf<int64_t> slice_ptr;  // first entry of each slice (n_slices + 1)
  DevBuf<int32_t> slice_w;    // width (entries per row) of each slice
  DevBuf<int32_t> sell_col;   // packed (signed) column indices
  DevBuf<double> sell_val;    // kSell only
  double scale = 1.0;         // kSigned: |value|
  bool ell = false;           // narrow operator stored as plain ELL (width ell_w)
  int ell_w = 0;
  // launch k_ell / k_sell_pipe as programmatic dependents (set per handle:
  // SFEEC_PDL read once at creation; off in the multi-rank paths)
  bool pdl = true;
  void upload(const HostCSR& h, bool strict_only, cudaStream_t s);
  // production layouts make the CSR copy redundant: free it (halves the
  // footprint of Q_sym at 256^3); has_csr() tells export paths
  void drop_csr() {
    rp.reset();
    ci.reset();
    val.reset();
  }
  bool has_csr() const { return rp.p != nullptr; }
  // production layout built on the device from a device CSR (same layout
  // decisions as upload(); only the row pointers visit the host); the CSR
  // buffers are consumed
  void upload_device(DevCSR&& d, cudaStream_t s);
  // keep a device CSR as is (CSR-vector kernel)
  void adopt_csr(DevCSR&& d) {
    rows = d.rows;
    cols = d.cols;
    nnz = d.nnz;
    rp = std::move(d.rp);
    ci = std::move(d.ci);
    val = std::move(d.val);
    const double avg = rows ? (double)nnz / (double)rows : 0.0;
    tpr = 1;
    while (tpr < 32 && tpr * 2 <= avg) tpr *= 2;
    layout = kCsr;
  }
  void download_csr(int64_t* row_ptr, int32_t* col_idx, double* v, cudaStream_t s) const;
  // algorithmic bytes of one application in this layout (arrays streamed once)
  double stream_bytes() const;
};

void launch_spmv_strict(const DevOperator& a, const double* x, double* y, cudaStream_t s);
void launch_spmv_axpy_strict(const DevOperator& a, const double* x, double* y, double alpha,
                             cudaStream_t s);
// accumulate ? y += alpha * A x : y = A x
void launch_spmv(const DevOperator& a, const double* x, double* y, double alpha,
                 bool accumulate, cudaStream_t s);
// y += alpha * x   (strict: y + (alpha*x) with separate rounding)
void launch_axpy(double* y, const double* x, double alpha, int64_t n, bool strict,
                 cudaStream_t s);
// x = y / nrm
void launch_scale_copy(double* x, const double* y, double inv, double nrm, int64_t n,
                       cudaStream_t s);

}  // namespace sfeec_b200
