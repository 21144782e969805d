// Exception -> ew_status translation shared by the C ABI translation units:
// every entry point runs its C++ body inside guarded(), so nothing throws
// across the boundary and ew_last_error() carries the message.
#pragma once

#include <stdexcept>
#include <string>

#include "elaskit/communicator.hpp"
#include "elaskit/dataflow.hpp"
#include "elaskit/device.hpp"
#include "elaskit/migration.hpp"
#include "elaskit/param_fabric.hpp"
#include "elaskit/rng.hpp"
#include "ew_api.h"

namespace ew {

int set_error(int status, const std::string& msg);

template <class F>
inline int guarded(F&& body) {
  try {
    return body();
  } catch (const elaskit::CoverageMismatch& e) {
    return set_error(EW_ERR_COVERAGE_MISMATCH, e.what());
  } catch (const elaskit::MissingBackup& e) {
    return set_error(EW_ERR_MISSING_BACKUP, e.what());
  } catch (const elaskit::NoSurvivors& e) {
    return set_error(EW_ERR_NO_SURVIVORS, e.what());
  } catch (const elaskit::DimensionMismatch& e) {
    return set_error(EW_ERR_DIMENSION_MISMATCH, e.what());
  } catch (const elaskit::MismatchedDpDegree& e) {
    return set_error(EW_ERR_MISMATCHED_DP, e.what());
  } catch (const elaskit::DisconnectedGroup& e) {
    return set_error(EW_ERR_DISCONNECTED, e.what());
  } catch (const elaskit::InsufficientTargetMemory& e) {
    return set_error(EW_ERR_INSUFFICIENT_MEMORY, e.what());
  } catch (const elaskit::device::CudaError& e) {
    return set_error(EW_ERR_CUDA, e.what());
  } catch (const std::invalid_argument& e) {
    return set_error(EW_ERR_INVALID_ARGUMENT, e.what());
  } catch (const std::out_of_range& e) {
    return set_error(EW_ERR_OUT_OF_RANGE, e.what());
  } catch (const std::exception& e) {
    return set_error(EW_ERR_INTERNAL, e.what());
  } catch (...) {
    return set_error(EW_ERR_INTERNAL, "unknown exception");
  }
}

}  // namespace ew
