# Build the sm_100a C-ABI library and the CPU oracle.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v -Iinclude
SRC := $(wildcard paper_1211_1680_b200/csrc/*.cu)
HDR := $(wildcard paper_1211_1680_b200/csrc/*.cuh paper_1211_1680_b200/csrc/*.h paper_1211_1680_b200/csrc/*.inc) include/s2w.h
LIB := paper_1211_1680_b200/lib/libs2w.so
OBJ := $(patsubst paper_1211_1680_b200/csrc/%.cu,build/%.o,$(SRC))

all: $(LIB) oracle

build/%.o: paper_1211_1680_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJ)
	@mkdir -p paper_1211_1680_b200/lib
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart_static -lrt -lpthread -ldl

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
