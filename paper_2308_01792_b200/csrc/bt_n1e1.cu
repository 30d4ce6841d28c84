// Nédélec N1E1 curl-curl + mass operator (no reference implementation;
// SPEC.md:8). Placeholder entry points until the kernel lands.
#include "bt_internal.hpp"

extern "C" {
bt_status bt_n1e1_create(const bt_grid*, int, double, double, bt_n1e1**) {
  bt::set_error("N1E1 operator not built in this version");
  return BT_LOGIC_ERROR;
}
void bt_n1e1_destroy(bt_n1e1*) {}
bt_status bt_apply_n1e1(const bt_n1e1*, const double*, double*, int, void*) {
  bt::set_error("N1E1 operator not built in this version");
  return BT_LOGIC_ERROR;
}
bt_status bt_n1e1_sync(const bt_grid*, int, double*, void*) {
  bt::set_error("N1E1 operator not built in this version");
  return BT_LOGIC_ERROR;
}
}
