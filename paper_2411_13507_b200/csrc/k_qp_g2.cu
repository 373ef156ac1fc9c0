// Cut-QP kernels and launcher for gamma = 2 (see k_qp_impl.cuh).
#define BZG_QP_G 2
#include "k_qp_impl.cuh"
