# Build the product library (sm_100a) and the test-only oracle.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG := paper_2111_10270_b200
SRC := $(PKG)/csrc/plan.cpp $(PKG)/csrc/solver.cpp $(PKG)/csrc/kernels.cu $(PKG)/csrc/compile_gpu.cu
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -v -Iinclude -I$(PKG)/csrc

all: $(PKG)/libfastdog.so oracle/liboracle.so

$(PKG)/libfastdog.so: $(SRC) $(PKG)/csrc/internal.h include/fastdog.h
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) -ldl 2> build_ptxas.log || (cat build_ptxas.log; false)

oracle/liboracle.so: oracle/oracle.c oracle/oracle.h
	gcc -O2 -std=c11 -fopenmp -fPIC -shared -Wall -o $@ oracle/oracle.c -lm

clean:
	rm -f $(PKG)/libfastdog.so oracle/liboracle.so build_ptxas.log

.PHONY: all clean
