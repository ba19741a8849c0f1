// Reference header name (/root/reference/proj/include/tdp/timing_graph.hpp) -> the B200 drop-in API.
#pragma once
#include "tdp/tdp_api.hpp"
