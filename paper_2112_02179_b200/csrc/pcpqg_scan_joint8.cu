// Instantiations of the scan kernel for one family of code layouts.
#include "pcpqg_scan.cuh"

namespace pcpqg {
ScanFn scan_fn_joint8(bool k16, int nq) { return k16 ? pick_nq<0, 0, 16>(nq) : pick_nq<0, 0>(nq); }
}  // namespace pcpqg
