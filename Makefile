# Builds the sm_100a CUDA library (the product) and the CPU oracle (test-only).
NVCC     ?= nvcc
CC       ?= gcc
PKG      := paper_2109_08219_b200
LIB      := $(PKG)/_lib/libdtopk.so
SRCS     := $(PKG)/csrc/api.cu
HDRS     := $(wildcard $(PKG)/csrc/*.cuh) include/dtopk.h
NVFLAGS  := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
            -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr -Xptxas -v
ORACLE   := oracle/_build/libdtopk_oracle.so

all: $(LIB) $(ORACLE)

$(LIB): $(SRCS) $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) 2> $(PKG)/_lib/ptxas.log || (cat $(PKG)/_lib/ptxas.log; exit 1)

$(ORACLE): oracle/dtopk_oracle.c oracle/dtopk_oracle.h
	@mkdir -p $(dir $@)
	$(CC) -O3 -march=native -fPIC -shared -pthread -o $@ oracle/dtopk_oracle.c

sass: $(LIB)
	cuobjdump -sass $(LIB) > $(PKG)/_lib/libdtopk.sass

clean:
	rm -rf $(PKG)/_lib oracle/_build

.PHONY: all clean sass
