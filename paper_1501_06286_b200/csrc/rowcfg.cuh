// rowcfg.cuh — compile-time configuration of the row kernel (K1).
#pragma once
// points per thread of the register row FFT (8 or 16)
#ifndef QMC_ROW_E
#define QMC_ROW_E 16
#endif
// minimum CTAs per SM requested from ptxas for K1 (register budget)
#ifndef QMC_ROWS_MINB
#define QMC_ROWS_MINB 2
#endif
// ... for K1 CTAs of 512 or more threads
#ifndef QMC_ROWS_MINB512
#define QMC_ROWS_MINB512 1
#endif
