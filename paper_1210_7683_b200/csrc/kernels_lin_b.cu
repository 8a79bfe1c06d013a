// kernels_lin_b.cu — split-grid linear-solve kernel instantiations for p in [17, 32].
#include "linear_solve.cuh"

namespace gwg {

bool lin_ops_for_b(int64_t p, LinOps* out) {
  switch (p) {
    case 17:
      *out = make_lin_ops<17>();
      return true;
    case 18:
      *out = make_lin_ops<18>();
      return true;
    case 19:
      *out = make_lin_ops<19>();
      return true;
    case 20:
      *out = make_lin_ops<20>();
      return true;
    case 21:
      *out = make_lin_ops<21>();
      return true;
    case 22:
      *out = make_lin_ops<22>();
      return true;
    case 23:
      *out = make_lin_ops<23>();
      return true;
    case 24:
      *out = make_lin_ops<24>();
      return true;
    case 25:
      *out = make_lin_ops<25>();
      return true;
    case 26:
      *out = make_lin_ops<26>();
      return true;
    case 27:
      *out = make_lin_ops<27>();
      return true;
    case 28:
      *out = make_lin_ops<28>();
      return true;
    case 29:
      *out = make_lin_ops<29>();
      return true;
    case 30:
      *out = make_lin_ops<30>();
      return true;
    case 31:
      *out = make_lin_ops<31>();
      return true;
    case 32:
      *out = make_lin_ops<32>();
      return true;
    default:
      return false;
  }
}

}  // namespace gwg
