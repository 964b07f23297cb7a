// vv_host_common.h -- host-side shared state of the C ABI (error slot,
// basis-table constants).  Not part of the public header.
#pragma once
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

namespace vv {

// thread-local last error message (vv_last_error)
std::string &last_error();
int set_error(int code, const char *fmt, ...);

// Host restatement of kernels.basis_tables (kernels.py:56-76) through
// hh.hh_norm (hh.py:249-262) and hh._sh_prefactor (hh.py:193-207),
// float64, same operation order as the Python.
struct HostTables {
    int n_max, k, s, n_pairs;
    int64_t pair_n[64], pair_l[64], k2pair[256], k2sh[256];
    double pair_norm[64], sh_pref[128];
};
int build_tables(int n_max, HostTables &t);

}  // namespace vv
