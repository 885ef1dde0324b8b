// Instantiations of the scan kernel for one family of code layouts.
#include "pcpqg_scan.cuh"

namespace pcpqg {
ScanFn scan_fn_p16(uint32_t sw, int nq) {
  switch (sw) {
    case 0: return pick_nq<16, 0>(nq);
    case 4: return pick_nq<16, 4>(nq);
    case 8: return pick_nq<16, 8>(nq);
    case 16: return pick_nq<16, 16>(nq);
    case 32: return pick_nq<16, 32>(nq);
  }
  return nullptr;
}
}  // namespace pcpqg
