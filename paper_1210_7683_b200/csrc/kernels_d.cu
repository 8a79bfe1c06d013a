// kernels_d.cu — grid/prep kernel instantiations for p in [25, 32].
#include "kernel_table.cuh"

namespace gwg {

bool ops_for_d(int64_t p, KernelOps* out) {
  switch (p) {
    case 25:
      *out = make_ops<25>();
      return true;
    case 26:
      *out = make_ops<26>();
      return true;
    case 27:
      *out = make_ops<27>();
      return true;
    case 28:
      *out = make_ops<28>();
      return true;
    case 29:
      *out = make_ops<29>();
      return true;
    case 30:
      *out = make_ops<30>();
      return true;
    case 31:
      *out = make_ops<31>();
      return true;
    case 32:
      *out = make_ops<32>();
      return true;
    default:
      return false;
  }
}

}  // namespace gwg
