/* TEST INFRASTRUCTURE ONLY: host build of the product's glibc-exp
 * restatement (paper_1805_11007_b200/csrc/glibc_exp.h), so the CPU tests can
 * compare it with the host libm exp bit for bit. */
#include "../paper_1805_11007_b200/csrc/glibc_exp.h"
double cs_exp_host(double x) { return cs_exp(x); }
