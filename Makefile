# Build of the three shared libraries (all in-tree so they travel to the GPU box):
#   paper_1204_1533_b200/liblinedg_b200.so  -- sm_100a hot path + C-ABI (product)
#   paper_1204_1533_b200/liblinedg_host.so  -- setup library (basis/mesh/mapping/generators)
#   oracle/liblinedg_oracle.so              -- CPU oracle (test infrastructure only)
NVCC     ?= nvcc
# /usr/bin/g++ ships libgomp (OpenMP for the CPU oracle); the toolchain under /opt/gcc does not.
CXX      := $(shell test -x /usr/bin/g++ && echo /usr/bin/g++ || echo g++)
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := -std=c++17 $(ARCH) -lineinfo -O3 -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr \
            -diag-suppress 177
CXXFLAGS := -std=c++17 -O3 -march=x86-64-v3 -fPIC -Iinclude -Wall -Wno-unused-function

PKG      := paper_1204_1533_b200
CUDIR    := $(PKG)/csrc/cuda
HOSTDIR  := $(PKG)/csrc/host
OBJDIR   := build/obj

CU_SRCS  := $(wildcard $(CUDIR)/*.cu)
CU_OBJS  := $(patsubst $(CUDIR)/%.cu,$(OBJDIR)/cuda/%.o,$(CU_SRCS))
CU_HDRS  := $(wildcard $(CUDIR)/*.cuh) include/linedg_b200.h

all: $(PKG)/liblinedg_b200.so $(PKG)/liblinedg_host.so oracle/liblinedg_oracle.so

$(OBJDIR)/cuda/%.o: $(CUDIR)/%.cu $(CU_HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(PKG)/liblinedg_b200.so: $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart

$(PKG)/liblinedg_host.so: $(HOSTDIR)/linedg_host.cpp $(HOSTDIR)/lh_capi.cpp $(HOSTDIR)/linedg_host.hpp include/linedg_b200.h
	$(CXX) $(CXXFLAGS) -ffp-contract=off -shared -o $@ $(HOSTDIR)/linedg_host.cpp $(HOSTDIR)/lh_capi.cpp

oracle/liblinedg_oracle.so: oracle/oracle.cpp oracle/oracle_physics.hpp include/linedg_b200.h
	$(CXX) $(CXXFLAGS) -fopenmp -shared -o $@ oracle/oracle.cpp

# The reference's own setup sources against the Eigen shim (test infrastructure;
# skipped when /root/reference is absent).
ref:
	./oracle/ref_build/build.sh

clean:
	rm -rf build $(PKG)/*.so oracle/*.so

.PHONY: all clean ref

# Variant build for A/B timing (bench.py with LDG_B200_LIB=build/var/$(VAR)/liblinedg_b200.so):
#   make variant VAR=name VFLAGS="-DLDG_JT_SMALL=128 -DLDG_JT_MINB=6"
variant:
	@mkdir -p build/var/$(VAR)/obj
	for f in $(CU_SRCS); do $(NVCC) $(NVFLAGS) $(VFLAGS) -c $$f -o build/var/$(VAR)/obj/$$(basename $$f .cu).o & done; wait
	$(NVCC) $(ARCH) -shared -o build/var/$(VAR)/liblinedg_b200.so build/var/$(VAR)/obj/*.o -lcudart
	rm -rf build/var/$(VAR)/obj
