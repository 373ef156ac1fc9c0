// Cut-QP kernels and launcher for gamma = 1 (see k_qp_impl.cuh).
#define BZG_QP_G 1
#include "k_qp_impl.cuh"
