// Cut-QP kernels and launcher for gamma = 4 (see k_qp_impl.cuh).
#define BZG_QP_G 4
#include "k_qp_impl.cuh"
