// Co-residency build of the device code (MT_OPT_CTAS_PER_SM = 2): the same
// kernels compiled for two 128-thread CTAs per SM with a 96 KB conv ring each, in namespace mtk_cr
// (see mt_types.h).
#define MT_CR 1
#include "kernels.cu"
