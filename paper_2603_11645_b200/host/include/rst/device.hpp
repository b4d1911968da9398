// rst/device.hpp -- the device handle behind a host Graph.
//
// run_algorithm takes a const Graph& like the reference; the first call on
// a Graph uploads it (int64 -> int32 on the device) and later calls on the
// same unchanged Graph reuse the device copy and its workspace.
#pragma once

#include <string>

#include "rst/graph.hpp"
#include "rstg.h"

namespace rst {

// Device handle for g (cached per thread; re-uploaded if g changed).
rstg_graph* device_graph(const Graph& g, int device);
void drop_device_graphs();
// Throws the mapped exception type for a non-zero rstg status.
void rstg_check(int rc);

}  // namespace rst
