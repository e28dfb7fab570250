// ORACLE SHIM — test infrastructure only: main() for the reference's gtest files.
#include <gtest/gtest.h>

int main(int argc, char** argv) { return ::gts::run_all(argc, argv); }
