// Source-compatibility shim for reference include/ntf/tucker.hpp.
#pragma once
#include "ntf/ntf.hpp"
