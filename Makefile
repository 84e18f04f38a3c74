# Builds the in-tree C-ABI library paper_1802_05246_b200/libhermb200.so for sm_100a.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr
SRC := paper_1802_05246_b200/csrc
LIB := paper_1802_05246_b200/libhermb200.so
OBJ := build/capi.o build/tables.o

all: $(LIB) tools/fp64_peak

build/capi.o: $(SRC)/capi.cu $(wildcard $(SRC)/*.cuh) $(SRC)/tables.h include/hermb200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) $(PTXAS) -c $< -o $@

build/tables.o: $(SRC)/tables.cpp $(SRC)/tables.h
	@mkdir -p build
	g++ -O2 -fPIC -std=c++17 -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart

clean:
	rm -rf build $(LIB)

.PHONY: all clean tools

tools/fp64_peak: tools/fp64_peak.cu
	$(NVCC) $(ARCH) -O3 -o $@ $<

tools: tools/fp64_peak
