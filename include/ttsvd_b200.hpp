// ttsvd_b200.hpp — umbrella of the C++ drop-in for the reference's TT-SVD
// hot path on B200.  The per-header drop-ins live in include/ttsvd/ under the
// reference's own file names (errors, shape, storage, counters, threading,
// tsqr, small_svd, tsmm, tensor_train, tt_svd, perf_model, report), so a
// reference caller switches by pointing its include path at this
// repository's include/ instead of proj/include/ and linking
// -lttsvd_cu -lcudart; every numeric call runs on the GPU through the C-ABI
// of ttsvd_cu.h.
//
//   tsqr             tsqr.hpp:247        reduce_block       tsqr.hpp:208
//   combine_factors  tsqr.hpp:230        small_svd          small_svd.hpp:196
//   jacobi_svd       small_svd.hpp:120   select_rank        small_svd.hpp:49
//   derive_delta     small_svd.hpp:41    tsmm_reshape       tsmm.hpp:20, :74
//   transpose_reorder tsmm.hpp:90, :121  detail::run_chain  tt_svd.hpp:159
//   tt_svd_tsqr      tt_svd.hpp:281      tt_svd_distributed tt_svd.hpp:520
//   choose_combined_dims tt_svd.hpp:316  tt_svd_thick_bounds tt_svd.hpp:338
//   tt_svd_two_sided tt_svd.hpp:402      tt_svd_reference   tt_svd.hpp:215
#pragma once

#include "ttsvd/errors.hpp"
#include "ttsvd/shape.hpp"
#include "ttsvd/counters.hpp"
#include "ttsvd/threading.hpp"
#include "ttsvd/storage.hpp"
#include "ttsvd/tsqr.hpp"
#include "ttsvd/small_svd.hpp"
#include "ttsvd/tsmm.hpp"
#include "ttsvd/tensor_train.hpp"
#include "ttsvd/tt_svd.hpp"
#include "ttsvd/perf_model.hpp"
#include "ttsvd/report.hpp"
