// kernels_b.cu — grid/prep kernel instantiations for p in [9, 16].
#include "kernel_table.cuh"

namespace gwg {

bool ops_for_b(int64_t p, KernelOps* out) {
  switch (p) {
    case 9:
      *out = make_ops<9>();
      return true;
    case 10:
      *out = make_ops<10>();
      return true;
    case 11:
      *out = make_ops<11>();
      return true;
    case 12:
      *out = make_ops<12>();
      return true;
    case 13:
      *out = make_ops<13>();
      return true;
    case 14:
      *out = make_ops<14>();
      return true;
    case 15:
      *out = make_ops<15>();
      return true;
    case 16:
      *out = make_ops<16>();
      return true;
    default:
      return false;
  }
}

}  // namespace gwg
