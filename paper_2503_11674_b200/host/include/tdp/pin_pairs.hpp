// Reference header name (/root/reference/proj/include/tdp/pin_pairs.hpp) -> the B200 drop-in API.
#pragma once
#include "tdp/tdp_api.hpp"
