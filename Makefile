# Build every native artefact in-tree (the .so files travel to the GPU box with gpurun).
#   libgsg.so      -- the C-ABI CUDA library (sm_100a), paper_2010_03166_b200/
#   libgsgen.so    -- seeded workload generator (host C++), workload/
#   liboracle.so   -- fp64 CPU oracle (plain C, test infrastructure), oracle/
NVCC ?= /usr/local/cuda/bin/nvcc
CXX := /usr/bin/g++
CC := /usr/bin/gcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           --expt-relaxed-constexpr -Iinclude -Ipaper_2010_03166_b200/csrc
PKG := paper_2010_03166_b200
CSRC := $(wildcard $(PKG)/csrc/*.cu)
CHDR := $(wildcard $(PKG)/csrc/*.cuh) include/gsg.h
OBJS := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(CSRC))

all: gen oracle gsg

gen: workload/libgsgen.so
oracle: oracle/liboracle.so
gsg: $(PKG)/libgsg.so

workload/libgsgen.so: workload/csrc/gsgen.cpp
	$(CXX) -O2 -std=c++17 -fPIC -shared -o $@ $<

oracle/liboracle.so: oracle/oracle.c
	$(CC) -O2 -std=c11 -fPIC -shared -fopenmp -o $@ $< -lm

build/%.o: $(PKG)/csrc/%.cu $(CHDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -dc -o $@ $<

$(PKG)/libgsg.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -Xcompiler -fPIC -lcudart_static -ldl -lrt -lpthread

clean:
	rm -rf build workload/libgsgen.so oracle/liboracle.so $(PKG)/libgsg.so

.PHONY: all gen oracle gsg clean
