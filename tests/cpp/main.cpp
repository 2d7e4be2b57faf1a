#include "check.hpp"
int main(int argc, char** argv) { return check::run_all(argc, argv); }
