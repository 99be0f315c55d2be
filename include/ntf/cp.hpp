// Source-compatibility shim for reference include/ntf/cp.hpp.
#pragma once
#include "ntf/ntf.hpp"
