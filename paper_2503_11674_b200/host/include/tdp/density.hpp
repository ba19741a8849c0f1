// Reference header name (/root/reference/proj/include/tdp/density.hpp) -> the B200 drop-in API.
#pragma once
#include "tdp/tdp_api.hpp"
