// Instantiations of the scan kernel for one family of code layouts.
#include "pcpqg_scan.cuh"

namespace pcpqg {
ScanFn scan_fn_joint8(bool k16, int nq) { return k16 ? pick_nq<0, 0, 16>(nq) : pick_nq<0, 0>(nq); }

// filter mode (fp16 pre-score + exact re-score), k = 16, groups of 16
ScanFn scan_fn_joint8_filter() { return scan_topk_kernel<16, 0, 0, 16, false, true>; }

// pre-multiplied eta*lambda table, small query groups only
ScanFn scan_fn_joint8_table(int nq) {
  switch (nq) {
    case 1: return scan_topk_kernel<1, 1, 0, 0>;
    case 2: return scan_topk_kernel<2, 1, 0, 0>;
    case 1 | kWsFlag: return scan_topk_kernel<1, 1, 0, 0, true>;
    case 2 | kWsFlag: return scan_topk_kernel<2, 1, 0, 0, true>;
  }
  return nullptr;
}
}  // namespace pcpqg
