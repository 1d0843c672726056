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
struct StencilOp;

// Column-delta forms of both layouts (SFEEC_DELTA=1; off by default, measured
// slower: spmv_kernels.cu delta_enabled). Inside a slice (or a 32-row ELL group) entry k of lane l sits at
// column base_sel[k] + l + delta: two int32 bases per (slice, entry), read by
// the whole warp as broadcasts, plus a uint16 code per entry (sel bit + delta,
// kSigned: sel + delta + negative bit). The tet numbering puts consecutive
// rows at neighbouring vertices of one entity type, so the k-th neighbours of
// a slice's rows are consecutive ids; the second base covers slices that
// straddle two types. 10.1 B/entry instead of 12 (values), 2.1 instead of 4
// (incidence). A slice whose codes do not fit keeps int32 columns ("full").
// Codes are stored in chunks of 4 entries per lane (one 8-byte load per lane
// per chunk).
// Windowed sliced layout ("win", the default where it fits): the rows are cut
// into units of whole slices (~1-2k rows); the columns a unit touches, in
// 32-column blocks, form its window (a few contiguous id ranges: the k-major
// numbering puts a row's neighbours in 3 vertex planes x 3 vertex rows). A
// persistent CTA per SM stages each unit's window of x in shared memory with
// bulk async copies (cp.async.bulk, mbarrier completion; double-buffered, a
// producer warp runs one unit ahead) while 8 consumer warps stream the
// unit's slices: fp64 values plus a uint16 window index per entry (kSigned:
// index << 1 | negative) -- 10 B/entry (values) or 2 B/entry (incidence)
// instead of 12 / 4 -- and gather x from shared memory instead of L2.
struct WUnit {
  int64_t s0;       // first slice
  int32_t ns;       // slices
  int32_t seg0;     // first segment
  int32_t nseg;     // segments
  int32_t wsize;    // window size (doubles, a multiple of 32)
  int32_t pad[2];
};
// segment: window columns [col, col + len) land at shared index dst, len =
// next dst - dst (the unit's wsize for its last segment)
constexpr int kWinCap = 14336;  // doubles per window buffer (112 KB)

struct DSlice {
  int64_t r0;    // first row
  int64_t vptr;  // first value (entry k of lane l at vptr + k*nr + l)
  int64_t dptr;  // first int16 of the deltas (or of the int32 columns of a full slice)
  int32_t bptr;  // first base column (4-aligned)
  int32_t nw;    // w | nr << 20 | full << 26
};

struct DevOperator {
  // kStencil: mesh-aware layout of the device-assembled tet operators
  // (stencil.cuh): column ids recomputed from the Kuhn stencil, values only
  enum Layout { kCsr = 0, kSigned = 1, kSell = 2, kStencil = 3 };
  std::shared_ptr<StencilOp> st;
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
  // column-delta form (see DSlice): sliced -> dslice; ELL -> 32-row groups,
  // group g's bases at dbase[g*W4], deltas at dcol[g*32*W4], values at
  // sell_val[g*32*W], dfull[g] = index of its int32 columns in sell_col or -1
  bool delta = false;
  int64_t n_full = 0;  // slices / groups that kept int32 columns
  DevBuf<DSlice> dslice;
  DevBuf<int32_t> dbase;
  DevBuf<uint16_t> dcol;
  DevBuf<int32_t> dfull;
  // windowed layout (see WUnit): dslice (codes at dptr, chunks of 8 entries
  // per lane), dcol, sell_val, plus the units and their segments
  bool win = false;
  int64_t n_units = 0;
  int64_t win_rows = 0;   // target rows per unit the build settled on
  bool win_narrow = false;  // every slice <= 8 wide: codes entry-major, no chunks
  DevBuf<WUnit> wunit;
  DevBuf<int2> wseg;      // {first column, shared index}

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
  // column-delta builders from a device CSR (kSell / kSigned decided)
  void build_dsell(const int64_t* rp, const int32_t* ci, const double* v,
                   const std::vector<int64_t>& hrow, const std::vector<int32_t>& hw,
                   cudaStream_t s);
  void build_dell(const int64_t* rp, const int32_t* ci, const double* v, int w, cudaStream_t s);
  // windowed layout from a device CSR; false (nothing changed) when some
  // unit's window cannot fit kWinCap even at the smallest unit size
  bool build_win(const int64_t* rp, const int32_t* ci, const double* v,
                 const std::vector<int64_t>& hrow, const std::vector<int32_t>& hw,
                 cudaStream_t s);
};

// the windowed kernel (window_spmv.cu)
void launch_win(const DevOperator& a, const double* x, double* y, double alpha, bool accumulate,
                cudaStream_t s);
bool win_enabled();
// the TMA-streamed sliced kernel (stream_spmv.cu; fp64 sliced operators)
void launch_sell_tma(const DevOperator& a, const double* x, double* y, double alpha,
                     bool accumulate, cudaStream_t s);
bool sell_tma_enabled();
void prepare_sell_tma();

// Fused producer -> consumer pair (wave.cu): t = P x, then y += alpha C t in
// one persistent wavefront kernel (P sliced or ELL fp64, C ELL). A plan is
// built once per operator pair; ok == false means the layouts are not
// supported and the caller runs the two kernels.
struct WavePlan {
  bool built = false, ok = false;
  DevBuf<int4> items;
  int n_items = 0;
  int64_t n_prod = 0;
  DevBuf<int> sync;  // ticket + per-producer-item flags, cleared per launch
  unsigned grid = 0;
  int batch = 1;  // items per ticket
  void* kernel = nullptr;
};
bool wave_enabled();  // SFEEC_WAVE=1 (default off: measured slower, wave.cu)
bool build_wave_plan(const DevOperator& p, const DevOperator& c, WavePlan& plan, cudaStream_t s);
void launch_wave(const WavePlan& plan, const DevOperator& p, const DevOperator& c,
                 const double* x, double* t, double* y, double alpha, cudaStream_t s);

void launch_spmv_strict(const DevOperator& a, const double* x, double* y, cudaStream_t s);
void launch_spmv_axpy_strict(const DevOperator& a, const double* x, double* y, double alpha,
                             cudaStream_t s);
// accumulate ? y += alpha * A x : y = A x
// reverse: rows in descending order (k_ell, k_sell_pipe), so a kernel starts
// on the rows the previous kernel wrote last (still in L2); results unchanged
void launch_spmv(const DevOperator& a, const double* x, double* y, double alpha,
                 bool accumulate, cudaStream_t s, bool reverse = false);
// y += alpha * x   (strict: y + (alpha*x) with separate rounding)
void launch_axpy(double* y, const double* x, double alpha, int64_t n, bool strict,
                 cudaStream_t s);
// x = y / nrm
void launch_scale_copy(double* x, const double* y, double inv, double nrm, int64_t n,
                       cudaStream_t s);

}  // namespace sfeec_b200
