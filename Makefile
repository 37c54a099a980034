# Build the product library (sm_100a) and the test-only oracle.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG := paper_2111_10270_b200
SRC := $(PKG)/csrc/plan.cpp $(PKG)/csrc/solver.cpp $(PKG)/csrc/kernels.cu $(PKG)/csrc/compile_gpu.cu \
       $(PKG)/csrc/pack_gpu.cu
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -v -Iinclude -I$(PKG)/csrc

all: $(PKG)/libfastdog.so oracle/liboracle.so

OBJ := $(patsubst $(PKG)/csrc/%,build/obj/%.o,$(SRC))

# (make -j: the four sources compile concurrently; no --split-compile, which
# made ptxas's output vary from build to build)
build/obj/%.cu.o: $(PKG)/csrc/%.cu $(PKG)/csrc/internal.h include/fastdog.h
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; false)

build/obj/%.cpp.o: $(PKG)/csrc/%.cpp $(PKG)/csrc/internal.h include/fastdog.h
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(PKG)/libfastdog.so: $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -ldl
	@cat build/obj/*.ptxas.log > build_ptxas.log 2>/dev/null || true

oracle/liboracle.so: oracle/oracle.c oracle/oracle.h
	gcc -O2 -std=c11 -fopenmp -fPIC -shared -Wall -o $@ oracle/oracle.c -lm

clean:
	rm -rf $(PKG)/libfastdog.so oracle/liboracle.so build_ptxas.log build/obj

.PHONY: all clean
