# Builds the in-tree C-ABI library paper_1802_05246_b200/libhermb200.so for sm_100a.
# The eight 2D kernel orders live in separate translation units (kern_m*.cu)
# so `make -j` compiles them in parallel.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr
CXXFLAGS := -O2 -fPIC -std=c++17
SRC := paper_1802_05246_b200/csrc
LIB ?= paper_1802_05246_b200/libhermb200.so
BUILD ?= build
HDRS := $(wildcard $(SRC)/*.cuh) $(wildcard $(SRC)/*.h) include/hermb200.h
KERN := $(patsubst $(SRC)/%.cu,$(BUILD)/%.o,$(wildcard $(SRC)/kern_m*.cu))
OBJ := $(BUILD)/capi.o $(BUILD)/tables.o $(BUILD)/cellmap.o $(KERN)

all: $(LIB)

$(BUILD)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) $(PTXAS) $(EXTRA) -c $< -o $@

$(BUILD)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(BUILD)
	g++ $(CXXFLAGS) $(EXTRA) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart

clean:
	rm -rf build $(LIB)

.PHONY: all clean tools

# probe tools link the shared cudart (no static runtime copied into the tree)
tools/fp64_peak: tools/fp64_peak.cu
	$(NVCC) $(ARCH) -O3 -cudart shared -o $@ $<

tools: tools/fp64_peak
