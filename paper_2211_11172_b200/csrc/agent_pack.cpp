// Agent parameters and Adam moments between the reference's numpy lists and
// the device's flat fp64 layout (host C++).
//
// The drop-in hands the session's agent (rlcore.py:80-160: PolicyNet and
// ValueNet weight lists, the two Adam states' m and v, rlcore.py:50-71) to
// the device before every episode and writes the trained values back after
// it (tuner.py:350-440 updates them in place through ppo_update).  The
// flat layout (DeviceAgent._views) is the numpy arrays concatenated, except
// the tiling head, stored compact: only its legal columns (space.py
// head_columns).  A copy plan lists, per array, where its rows go:
//   flat[off + r*flat_ld + c] <-> host[r*host_ld + (cols ? cols[c] : c)]
// for r < rows, c < ncols -- contiguous arrays are one row, the tiling
// head's W and b gather/scatter through the column list.  One call runs the
// whole plan (three of them per direction: parameters, m, v), replacing
// ~20 numpy copies per list.
#include <cstdint>
#include <cstring>

#include "harl_b200.h"

extern "C" {

int harl_agent_copy(const harl_copy_op* ops, int32_t n_ops, double* flat,
                    int32_t to_host) {
  if (!ops || n_ops < 0 || !flat) return -1;
  if (to_host == 2) {   // compare only: 0 if every element is bitwise equal
    for (int32_t i = 0; i < n_ops; ++i) {
      const harl_copy_op& o = ops[i];
      if (!o.host || o.rows < 0 || o.ncols < 0 || o.off < 0) return -1;
      const double* h = static_cast<const double*>(o.host);
      const double* f = flat + o.off;
      for (int64_t r = 0; r < o.rows; ++r) {
        const double* fr = f + r * o.flat_ld;
        const double* hr = h + r * o.host_ld;
        if (!o.cols) {
          if (memcmp(hr, fr, (size_t)o.ncols * 8)) return 1;
        } else {
          for (int64_t c = 0; c < o.ncols; ++c)
            if (memcmp(&hr[o.cols[c]], &fr[c], 8)) return 1;
        }
      }
    }
    return 0;
  }
  for (int32_t i = 0; i < n_ops; ++i) {
    const harl_copy_op& o = ops[i];
    if (!o.host || o.rows < 0 || o.ncols < 0 || o.off < 0) return -1;
    double* h = static_cast<double*>(o.host);
    double* f = flat + o.off;
    for (int64_t r = 0; r < o.rows; ++r) {
      double* fr = f + r * o.flat_ld;
      double* hr = h + r * o.host_ld;
      if (!o.cols) {
        if (to_host) memcpy(hr, fr, (size_t)o.ncols * 8);
        else memcpy(fr, hr, (size_t)o.ncols * 8);
      } else if (to_host) {
        for (int64_t c = 0; c < o.ncols; ++c) hr[o.cols[c]] = fr[c];
      } else {
        for (int64_t c = 0; c < o.ncols; ++c) fr[c] = hr[o.cols[c]];
      }
    }
  }
  return 0;
}

}  // extern "C"
