// main() of the reference-suite binary (GoogleTest's gtest_main role).
#include <gtest/gtest.h>

int main(int argc, char** argv) { return gtshim::run_all(argc, argv); }
