// Host build of csrc/numfmt.cuh for the CPU tests (tests/test_numfmt.py).
#include "../../paper_2504_03683_b200/csrc/numfmt.cuh"

extern "C" {
int nf_double(double v, char* out) { return nf::fmt_double(v, out); }
int nf_ns(int64_t hi, uint64_t lo, char* out) { return nf::fmt_ns_div1000(hi, lo, out); }
int nf_int_of_double(double v, char* out) { return nf::fmt_int_of_double(v, out); }
int nf_i128(int64_t hi, uint64_t lo, char* out) { return nf::fmt_i128(hi, lo, out); }
}
