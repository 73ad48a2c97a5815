# Builds librcseg_b200.so for sm_100a (B200).  Also driven by
# __graft_entry__.build().  -fmad=false keeps fp64 arithmetic in numpy's
# rounding order; -lineinfo maps ncu source pages.
NVCC ?= nvcc
PKG := paper_1403_0240_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
HDR := $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.h) include/rcb.h
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
LIB := $(PKG)/librcseg_b200.so
ARCH := -gencode arch=compute_100a,code=sm_100a
FLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -fmad=false -Xcompiler -fPIC,-ffp-contract=off \
         -Xptxas -v -Iinclude

all: $(LIB)

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(FLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart_static

clean:
	rm -rf build $(LIB)

.PHONY: all clean
