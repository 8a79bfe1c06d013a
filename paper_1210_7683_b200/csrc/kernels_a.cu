// kernels_a.cu — grid/prep kernel instantiations for p in [1, 8].
#include "kernel_table.cuh"

namespace gwg {

bool ops_for_a(int64_t p, KernelOps* out) {
  switch (p) {
    case 1:
      *out = make_ops<1>();
      return true;
    case 2:
      *out = make_ops<2>();
      return true;
    case 3:
      *out = make_ops<3>();
      return true;
    case 4:
      *out = make_ops<4>();
      return true;
    case 5:
      *out = make_ops<5>();
      return true;
    case 6:
      *out = make_ops<6>();
      return true;
    case 7:
      *out = make_ops<7>();
      return true;
    case 8:
      *out = make_ops<8>();
      return true;
    default:
      return false;
  }
}

}  // namespace gwg
