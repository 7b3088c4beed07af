# Build libpagedattn.so (sm_100a kernels + C ABI + host allocator) and the oracle.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVXFLAGS ?=
NVFLAGS := $(ARCH) $(NVXFLAGS) -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
PKG := paper_2309_06180_b200
SRC := $(PKG)/csrc
OBJS := $(SRC)/pa_attention.o $(SRC)/pa_prefill.o $(SRC)/pa_decode_tc.o $(SRC)/pa_tp.o $(SRC)/pa_cache.o $(SRC)/pa_probe.o $(SRC)/pa_api.o $(SRC)/pa_alloc.o
HDRS := $(SRC)/pa_common.cuh $(SRC)/pa_tc.cuh $(SRC)/pa_internal.h include/pa.h

all: $(PKG)/libpagedattn.so oracle/liboracle.so

$(SRC)/%.o: $(SRC)/%.cu $(HDRS)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $@.ptxas.txt || (cat $@.ptxas.txt; false)

$(SRC)/%.o: $(SRC)/%.cpp $(HDRS)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(PKG)/libpagedattn.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

oracle/liboracle.so: oracle/oracle.c
	gcc -O2 -std=c99 -fPIC -shared -fopenmp -ffp-contract=off -fno-fast-math $< -o $@ -lm

clean:
	rm -f $(SRC)/*.o $(SRC)/*.ptxas.txt $(PKG)/libpagedattn.so oracle/liboracle.so

.PHONY: all clean
