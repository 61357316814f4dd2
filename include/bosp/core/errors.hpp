// Drop-in for the reference header bosp/core/errors.hpp (/root/reference/proj/include/bosp/core/errors.hpp):
// the B200 build declares the same names, argument meaning and exception types in
// paper_2506_08355_b200/csrc/api.hpp (namespace bosp, inline namespace b200).  Reference
// callers compile unchanged with  -I include -I paper_2506_08355_b200/csrc  and link
// libbosp_b200.so (tests/test_compat.py).
#pragma once
#include "api.hpp"
