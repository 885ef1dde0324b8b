// Instantiations of the scan kernel for one family of code layouts.
#include "pcpqg_scan.cuh"

namespace pcpqg {
ScanFn scan_fn_p8(uint32_t sw, int nq) {
  switch (sw) {
    case 0: return pick_nq<8, 0>(nq);
    case 4: return pick_nq<8, 4>(nq);
    case 8: return pick_nq<8, 8>(nq);
    case 16: return pick_nq<8, 16>(nq);
    case 32: return pick_nq<8, 32>(nq);
  }
  return nullptr;
}

// filter mode (fp16 pre-score + exact re-score), 4-bit scale codes, groups of 4
ScanFn scan_fn_p8_filter() { return scan_topk_kernel<4, 8, 4, 0, false, true>; }
}  // namespace pcpqg
