// Instantiations of the scan kernel for one family of code layouts.
#include "pcpqg_scan.cuh"

namespace pcpqg {
ScanFn scan_fn_p4(uint32_t sw, bool k16, int nq) {
  if (k16 && sw == 16) return pick_nq<4, 16, 16>(nq);
  if (k16 && sw == 32) return pick_nq<4, 32, 16>(nq);
  if (k16 && sw == 8) return pick_nq<4, 8, 16>(nq);
  switch (sw) {
    case 4: return pick_nq<4, 4>(nq);
    case 8: return pick_nq<4, 8>(nq);
    case 16: return pick_nq<4, 16>(nq);
    case 32: return pick_nq<4, 32>(nq);
  }
  return nullptr;
}

// filter mode (fp16 pre-score + exact re-score), raw fp16 alpha, k = 16, groups of 16
ScanFn scan_fn_p4_raw16_filter() { return scan_topk_kernel<16, 4, 16, 16, false, true>; }
}  // namespace pcpqg
