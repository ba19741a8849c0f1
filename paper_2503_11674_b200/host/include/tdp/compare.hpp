// Reference header name (/root/reference/proj/include/tdp/compare.hpp) -> the B200 drop-in API.
#pragma once
#include "tdp/tdp_api.hpp"
