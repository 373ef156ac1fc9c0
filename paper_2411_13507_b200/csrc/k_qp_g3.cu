// Cut-QP kernels and launcher for gamma = 3 (see k_qp_impl.cuh).
#define BZG_QP_G 3
#include "k_qp_impl.cuh"
