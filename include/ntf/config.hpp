// Source-compatibility shim for reference include/ntf/config.hpp.
#pragma once
#include "ntf/ntf.hpp"
