// shim.hpp — the reference's C++ surface (helio::) plus the batched engine
// handle the drop-in exposes beside it.
#pragma once

#include "helio/placement.hpp"
#include "helio/scheduler.hpp"
#include "shim_engine.hpp"
