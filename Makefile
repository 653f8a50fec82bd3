# Builds the product library (CUDA, sm_100a only) and the test-only C objects.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC,-O3 -shared --expt-relaxed-constexpr
PKG := paper_2402_01816_b200
LIB := $(PKG)/libgns.so
SRCS := $(PKG)/csrc/gns.cu $(wildcard $(PKG)/csrc/*.cuh) include/gns.h

all: $(LIB) oracle/liboracle.so synth/libsynth.so

$(LIB): $(SRCS)
	$(NVCC) $(NVFLAGS) -o $@ $(PKG)/csrc/gns.cu

oracle/liboracle.so: oracle/oracle.c
	gcc -O2 -std=c11 -shared -fPIC -o $@ $<

synth/libsynth.so: synth/gen.c
	gcc -O2 -std=c11 -shared -fPIC -o $@ $<

# bounds-asserting build for the GPU tests (GNS_LIB=libgns_debug.so)
debug: $(PKG)/libgns_debug.so

$(PKG)/libgns_debug.so: $(SRCS)
	$(NVCC) $(NVFLAGS) -DGNS_DEBUG_BOUNDS -o $@ $(PKG)/csrc/gns.cu

# A/B build with the register network merges on (binary32 merge pass, K1 merge-path
# rounds of both key widths; measured no faster); tests/test_gpu_knobs.py
net: $(PKG)/libgns_net.so

$(PKG)/libgns_net.so: $(SRCS)
	$(NVCC) $(NVFLAGS) -DGNS_F2_NET=1 -DGNS_K1_NET=3 -o $@ $(PKG)/csrc/gns.cu

# phase-timing build for experiments (GNS_LIB=libgns_prof.so, tools/prof_merge.py)
prof: $(PKG)/libgns_prof.so

$(PKG)/libgns_prof.so: $(SRCS)
	$(NVCC) $(NVFLAGS) -DGNS_PROF -o $@ $(PKG)/csrc/gns.cu

ptxas: $(SRCS)
	$(NVCC) $(NVFLAGS) -Xptxas -v -o /tmp/gns_ptxas.so $(PKG)/csrc/gns.cu 2>&1 | grep -E "Function properties|registers|spill|Compiling entry" 

sass: $(LIB)
	/usr/local/cuda/bin/cuobjdump -sass $(LIB)

clean:
	rm -f $(LIB) oracle/liboracle.so synth/libsynth.so

.PHONY: all debug net prof ptxas sass clean
