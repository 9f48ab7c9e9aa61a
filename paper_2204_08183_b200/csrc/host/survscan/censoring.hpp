// survscan/censoring.hpp — IPCW weights of the reference API
// (/root/reference/proj/include/survscan/censoring.hpp:38-45).  The device
// engine estimates them per engine (per CV fold) on the host and uploads
// G(Y-); Engine::ipcw() returns the host copy in dataset (sorted) order.
#pragma once

#include <vector>

namespace survscan {

struct IpcwWeights {
  std::vector<double> u;  // 1 / G(Y_r-) on competing-event rows, else 0
  std::vector<double> g;  // G(Y_i-) for every row
};

}  // namespace survscan
