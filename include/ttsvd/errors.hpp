// ttsvd/errors.hpp — B200 drop-in for the reference's exception tree
// (errors.hpp:9-62).  Same class names and hierarchy, so `catch (const
// ttsvd::Error&)` and the specific catches of reference callers keep working;
// DeviceError (new) carries CUDA / exchange failures of the device path.
#pragma once

#include <stdexcept>
#include <string>

namespace ttsvd {

class Error : public std::runtime_error {
public:
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};

// one leaf per failure class of the reference, in its order
#define TTSVD_DECLARE_ERROR(Name) \
    class Name : public Error {   \
        using Error::Error;       \
    };
TTSVD_DECLARE_ERROR(LayoutError)          // reshape needs a copy (storage.hpp:134)
TTSVD_DECLARE_ERROR(AllocationError)      // memory budget (storage.hpp:22-26)
TTSVD_DECLARE_ERROR(DimensionMismatch)    // R.m != M.cols, mixed parts (tsqr.hpp:213, 233)
TTSVD_DECLARE_ERROR(DimensionError)       // n < m (tsqr.hpp:250-251)
TTSVD_DECLARE_ERROR(DegenerateDimension)  // d < 2 (tt_svd.hpp:283)
TTSVD_DECLARE_ERROR(ConvergenceError)     // 30 Jacobi sweeps (small_svd.hpp:113)
TTSVD_DECLARE_ERROR(ShapeError)           // TSMM / reorder shapes (tsmm.hpp:23-26, 94-95)
TTSVD_DECLARE_ERROR(PartitionMismatch)    // distributed slabs (tt_svd.hpp:523-526)
TTSVD_DECLARE_ERROR(DivergenceError)      // cost-model series (perf_model.hpp:119)
TTSVD_DECLARE_ERROR(IoError)              // files and reports
TTSVD_DECLARE_ERROR(DeviceError)          // CUDA / NCCL / exchange failure (B200 path only)
#undef TTSVD_DECLARE_ERROR

}  // namespace ttsvd
