// kernels_c.cu — grid/prep kernel instantiations for p in [17, 24].
#include "kernel_table.cuh"

namespace gwg {

bool ops_for_c(int64_t p, KernelOps* out) {
  switch (p) {
    case 17:
      *out = make_ops<17>();
      return true;
    case 18:
      *out = make_ops<18>();
      return true;
    case 19:
      *out = make_ops<19>();
      return true;
    case 20:
      *out = make_ops<20>();
      return true;
    case 21:
      *out = make_ops<21>();
      return true;
    case 22:
      *out = make_ops<22>();
      return true;
    case 23:
      *out = make_ops<23>();
      return true;
    case 24:
      *out = make_ops<24>();
      return true;
    default:
      return false;
  }
}

}  // namespace gwg
