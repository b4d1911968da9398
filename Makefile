# Build of the B200 RST engine. Everything is compiled for sm_100a only.
#   make            -> paper_2603_11645_b200/librstg.so (CUDA kernels + C ABI)
#                      paper_2603_11645_b200/librst_b200.so (C++ rst:: mirror)
#                      build/rst, build/rst_bench, build/rst_acceptance
#   make oracle     -> the checker (oracle/, test infrastructure only)
NVCC ?= nvcc
CXX ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall \
           --expt-relaxed-constexpr -Xptxas -v
PKG := paper_2603_11645_b200
CSRC := $(PKG)/csrc
OBJDIR := build/obj
CU := engine cc listrank tilerank euler euler_api pr bfs validate graph loader capi
OBJS := $(patsubst %,$(OBJDIR)/%.o,$(CU))
HDRS := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.hpp) include/rstg.h

HOST := $(PKG)/host
HOST_SRCS := $(wildcard $(HOST)/src/*.cpp)
CXXFLAGS := -std=c++20 -O2 -g -fPIC -Wall -I$(HOST)/include -Iinclude

all: $(PKG)/librstg.so $(PKG)/librst_b200.so build/rst build/rst_bench build/rst_acceptance

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.txt || (cat $(OBJDIR)/$*.ptxas.txt; false)

$(PKG)/librstg.so: $(OBJS)
	$(NVCC) $(ARCH) -shared $(OBJS) -o $@ -lcudart

$(PKG)/librst_b200.so: $(HOST_SRCS) $(wildcard $(HOST)/include/rst/*.hpp) $(PKG)/librstg.so
	$(CXX) $(CXXFLAGS) -shared $(HOST_SRCS) -o $@ -L$(PKG) -lrstg -Wl,-rpath,'$$ORIGIN' -lpthread

build/rst: $(HOST)/tools/rst_main.cpp $(PKG)/librst_b200.so
	@mkdir -p build
	$(CXX) $(CXXFLAGS) $< -o $@ -L$(PKG) -lrst_b200 -lrstg -Wl,-rpath,'$$ORIGIN/../$(PKG)'

build/rst_bench: $(HOST)/benchmarks/rst_bench.cpp $(PKG)/librst_b200.so
	@mkdir -p build
	$(CXX) $(CXXFLAGS) $< -o $@ -L$(PKG) -lrst_b200 -lrstg -Wl,-rpath,'$$ORIGIN/../$(PKG)'

build/rst_acceptance: $(HOST)/tests/acceptance.cpp $(PKG)/librst_b200.so
	@mkdir -p build
	$(CXX) $(CXXFLAGS) $< -o $@ -L$(PKG) -lrst_b200 -lrstg -Wl,-rpath,'$$ORIGIN/../$(PKG)'

# The reference's OWN acceptance suite (proj/tests/acceptance.cpp), compiled
# unchanged against the rst:: mirror headers and linked to the GPU library:
# built only where the reference sources exist (the binary travels to the box).
REF_TESTS ?= /root/reference/proj/tests
ifneq ($(wildcard $(REF_TESTS)/acceptance.cpp),)
all: build/ref_acceptance
build/ref_acceptance: $(REF_TESTS)/acceptance.cpp $(REF_TESTS)/oracles.hpp $(PKG)/librst_b200.so
	@mkdir -p build
	$(CXX) $(CXXFLAGS) -I$(REF_TESTS) $< -o $@ -L$(PKG) -lrst_b200 -lrstg -Wl,-rpath,'$$ORIGIN/../$(PKG)'
endif

lib: $(PKG)/librstg.so

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(PKG)/*.so

.PHONY: all lib oracle clean
