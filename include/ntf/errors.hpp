// Source-compatibility shim for reference include/ntf/errors.hpp.
#pragma once
#include "ntf/ntf.hpp"
