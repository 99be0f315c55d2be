// Source-compatibility shim for reference include/ntf/tensor.hpp.
#pragma once
#include "ntf/ntf.hpp"
