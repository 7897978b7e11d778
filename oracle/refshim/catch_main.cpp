// main() for the reference's Catch2 tests built against the shim (oracle/_ref).
#define CATCH_SHIM_MAIN
#include <catch2/catch_amalgamated.hpp>
