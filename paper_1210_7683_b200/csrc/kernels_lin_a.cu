// kernels_lin_a.cu — split-grid linear-solve kernel instantiations for p in [1, 16].
#include "linear_solve.cuh"
#include "grid_split.cuh"
namespace gwg {

// The S_BR launch of the split grid is p-independent.
SbrOps sbr_ops(int variant) {
  switch (variant) {
    case 1: return make_sbr_ops<SbrCfg<4, 5, 4, 1, 16, 5>>();
    case 2: return make_sbr_ops<SbrCfg<2, 5, 4, 1, 32, 4>>();
    default: return make_sbr_ops<SbrDefault>();
  }
}

bool lin_ops_for_a(int64_t p, LinOps* out) {
  switch (p) {
    case 1:
      *out = make_lin_ops<1>();
      return true;
    case 2:
      *out = make_lin_ops<2>();
      return true;
    case 3:
      *out = make_lin_ops<3>();
      return true;
    case 4:
      *out = make_lin_ops<4>();
      return true;
    case 5:
      *out = make_lin_ops<5>();
      return true;
    case 6:
      *out = make_lin_ops<6>();
      return true;
    case 7:
      *out = make_lin_ops<7>();
      return true;
    case 8:
      *out = make_lin_ops<8>();
      return true;
    case 9:
      *out = make_lin_ops<9>();
      return true;
    case 10:
      *out = make_lin_ops<10>();
      return true;
    case 11:
      *out = make_lin_ops<11>();
      return true;
    case 12:
      *out = make_lin_ops<12>();
      return true;
    case 13:
      *out = make_lin_ops<13>();
      return true;
    case 14:
      *out = make_lin_ops<14>();
      return true;
    case 15:
      *out = make_lin_ops<15>();
      return true;
    case 16:
      *out = make_lin_ops<16>();
      return true;
    default:
      return false;
  }
}

}  // namespace gwg
