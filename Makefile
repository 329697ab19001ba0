# Builds the in-tree C-ABI library paper_2603_16644_b200/libsklsq.so for sm_100a.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
SRC_DIR := paper_2603_16644_b200/csrc
SRCS := $(wildcard $(SRC_DIR)/*.cu)
OBJS := $(patsubst $(SRC_DIR)/%.cu,build/%.o,$(SRCS))
LIB := paper_2603_16644_b200/libsklsq.so

ORACLE_LIB := oracle/_build/liboracle.so

all: $(LIB) $(ORACLE_LIB)

oracle: $(ORACLE_LIB)

# the CPU oracle's compiled restatement (test infrastructure, never linked into the product)
$(ORACLE_LIB): oracle/csrc/*.c
	@mkdir -p oracle/_build
	gcc -O3 -fopenmp -ffp-contract=off -mavx2 -mf16c -fPIC -shared -o $@ oracle/csrc/*.c

build/%.o: $(SRC_DIR)/%.cu $(SRC_DIR)/*.cuh include/sklsq.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ > build/$*.ptxas.log 2>&1 || (cat build/$*.ptxas.log; exit 1)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -cudart static

clean:
	rm -rf build $(LIB) oracle/_build

.PHONY: all clean oracle
