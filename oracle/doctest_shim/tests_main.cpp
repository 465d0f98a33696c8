// main() of the doctest shim (test infrastructure).
#define DOCTEST_SHIM_MAIN
#include "doctest.h"
