# Top-level build: every native artefact, in-tree (the .so files travel to the GPU box with the
# repo snapshot).  `python -c "import __graft_entry__ as g; g.build()"` runs `make -j`.
PKG      := paper_2605_00429_b200
LIBDIR   ?= $(PKG)/lib
HOSTSRC  := $(wildcard $(PKG)/csrc/host/*.cpp)
HOSTHDR  := $(wildcard $(PKG)/csrc/host/*.hpp) include/p2m.h
CUDADIR  ?= $(PKG)/csrc/cuda
CUDASRC  := $(wildcard $(CUDADIR)/*.cu)
CUDAHDR  := $(wildcard $(CUDADIR)/*.cuh) include/p2m.h
NVCC     ?= /usr/local/cuda/bin/nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
# fp64 parity: no contraction anywhere on the distance path
CXXFLAGS := -O2 -g -std=gnu++17 -fPIC -ffp-contract=off -fvisibility=hidden -pthread -Wall -Wno-unused-function
NVFLAGS  := -O3 -std=c++17 $(ARCH) -lineinfo --fmad=false -Xcompiler -fPIC,-ffp-contract=off,-fvisibility=hidden \
            -Xptxas -v --expt-relaxed-constexpr $(NVEXTRA)

all: $(LIBDIR)/libp2m_host.so $(LIBDIR)/libp2m_cuda.so oracle examples/query_demo

$(LIBDIR)/libp2m_host.so: $(HOSTSRC) $(HOSTHDR)
	@mkdir -p $(LIBDIR)
	g++ $(CXXFLAGS) -shared -o $@ $(HOSTSRC)

$(LIBDIR)/libp2m_cuda.so: $(CUDASRC) $(CUDAHDR) $(LIBDIR)/libp2m_host.so
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(CUDASRC) -L$(LIBDIR) -lp2m_host -Xlinker -rpath,'$$ORIGIN' \
	    2> $(LIBDIR)/ptxas.log || (cat $(LIBDIR)/ptxas.log; false)

oracle:
	$(MAKE) -C oracle

clean:
	rm -f $(LIBDIR)/*.so
	$(MAKE) -C oracle clean

.PHONY: all oracle clean

examples/query_demo: examples/query_demo.cpp include/p2m_engine.hpp include/p2m.h $(LIBDIR)/libp2m_host.so $(LIBDIR)/libp2m_cuda.so
	g++ -O2 -std=c++17 -Iinclude -o $@ $< -L$(LIBDIR) -lp2m_cuda -lp2m_host -Wl,-rpath,'$$ORIGIN/../$(LIBDIR)'
