// Source-compatibility shim for reference include/ntf/divergence.hpp.
#pragma once
#include "ntf/ntf.hpp"
