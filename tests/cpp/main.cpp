// Test driver for the doctest-style C++ suites (tests/cpp/doctest.h).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"
