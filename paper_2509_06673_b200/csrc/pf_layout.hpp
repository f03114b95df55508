// pf_layout.hpp — storage layout of the factor values L of one supernode
// (host and device).
//
// A supernode with nc own columns and m rows (first nc rows = own columns)
// stores its strict-lower trapezoid in "panel-blocked" order: columns are cut
// into panels of kPW; each panel stores, as separate units,
//   1. its pw x pw unit-lower triangle, packed by rows (row ii holds
//      columns 0..ii-1 at ii(ii-1)/2), padded to an even count;
//   2. the rows below the panel in blocks of kRB rows, each block column-major
//      with its own row count nr (value (r, j) at j*nr + r), padded to even.
// Every unit is therefore a 16-byte multiple at a 16-byte aligned offset, so
// the sweep streams each one with a single TMA bulk copy, and consumes it in
// exactly the order it is stored (forward ascending, backward descending);
// the lane owning row r of a block reads consecutive shared-memory words and
// every per-lane triangle access is a base register plus an immediate.
#pragma once

#ifdef __CUDACC__
#define PF_HD __host__ __device__ __forceinline__
#else
#define PF_HD inline
#endif

namespace pf {

constexpr int kPW = 16;         // panel width (columns); even
constexpr int kRB = 32;         // rows per row block (one per lane)
constexpr int kMaxTaskSn = 64;  // supernodes per sweep task (task metadata lives in shared memory)

PF_HD int imin_(int a, int b) { return a < b ? a : b; }
PF_HD int even_up(int v) { return (v + 1) & ~1; }
PF_HD int tri_pad(int w) { return even_up(w * (w - 1) / 2); }

/// offset of the first value of panel p (all earlier panels are full width,
/// and full-width units need no padding because kPW is even)
PF_HD long long panel_base(int m, int p) {
  return (long long)p * tri_pad(kPW) + (long long)kPW * ((long long)p * m - (long long)kPW * p * (p + 1) / 2);
}

/// values of the rows-below part of a panel of width pw with nb rows below
PF_HD long long rows_size(int pw, int nb) {
  const int full = nb / kRB, rest = nb - full * kRB;
  return (long long)full * kRB * pw + even_up(rest * pw);
}

/// padded size of a supernode (values, even)
PF_HD long long sn_size(int nc, int m) {
  const int np = (nc + kPW - 1) / kPW, p0 = (np - 1) * kPW, pw = nc - p0;
  return panel_base(m, np - 1) + tri_pad(pw) + rows_size(pw, m - p0 - pw);
}

/// offset of L(i, j), j < nc, j < i < m, inside the supernode
PF_HD long long blk_off(int nc, int m, int i, int j) {
  const int p = j / kPW, p0 = p * kPW, pw = imin_(kPW, nc - p0), jj = j - p0;
  const long long pb = panel_base(m, p);
  if (i < p0 + pw) {
    const int ii = i - p0;
    return pb + ii * (ii - 1) / 2 + jj;
  }
  const int rr = i - (p0 + pw), b = rr / kRB, nb = m - p0 - pw, nr = imin_(kRB, nb - kRB * b);
  return pb + tri_pad(pw) + (long long)kRB * pw * b + (long long)jj * nr + (rr - kRB * b);
}

}  // namespace pf
