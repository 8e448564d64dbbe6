# Build the csconn C-ABI library for B200 (sm_100a) in-tree.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v $(EXTRA)
SRC := $(wildcard paper_2303_03279_b200/csrc/*.cu)
HDR := $(wildcard paper_2303_03279_b200/csrc/*.cuh) include/csconn.h
LIB := paper_2303_03279_b200/libcsconn.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build/ptxas.log || (cat build/ptxas.log; false)

$(SRC): | build
build:
	mkdir -p build

clean:
	rm -f $(LIB)

.PHONY: all clean
