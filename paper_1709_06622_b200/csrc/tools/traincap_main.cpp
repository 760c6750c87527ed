// `traincap` executable (reference: /root/reference/proj/tools/main.cpp).
#include "traincap/api.hpp"

int main(int argc, char** argv) { return traincap::run_cli(argc, argv); }
