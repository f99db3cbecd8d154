# Builds the three native artefacts (all in-tree so they travel to the GPU box):
#   paper_1307_6305_b200/lib/libamg_b200.so  -- the product (sm_100a CUDA + host driver, C ABI include/amg.h)
#   oracle/liboracle.so                       -- CPU oracle (test infrastructure only)
#   inputs/libgen.so                          -- seeded input generators (shared by tests and bench)
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
LIB := paper_1307_6305_b200/lib/libamg_b200.so
SRCS := paper_1307_6305_b200/csrc/driver.cu paper_1307_6305_b200/csrc/k_solve.cu paper_1307_6305_b200/csrc/k_dense.cu paper_1307_6305_b200/csrc/k_setup.cu paper_1307_6305_b200/csrc/k_tail.cu paper_1307_6305_b200/csrc/comm.cu paper_1307_6305_b200/csrc/dist.cu
OBJS := $(patsubst paper_1307_6305_b200/csrc/%.cu,build/%.o,$(SRCS))
HDRS := paper_1307_6305_b200/csrc/amg_internal.h paper_1307_6305_b200/csrc/hierarchy.h include/amg.h

all: $(LIB) oracle/liboracle.so inputs/libgen.so

build/%.o: paper_1307_6305_b200/csrc/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p paper_1307_6305_b200/lib
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -ldl

oracle/liboracle.so: oracle/amg_oracle.c
	gcc -O2 -std=c11 -D_DEFAULT_SOURCE -ffp-contract=off -fPIC -shared -o $@ $< -lm

inputs/libgen.so: inputs/gen.c
	gcc -O2 -std=c11 -D_DEFAULT_SOURCE -fPIC -shared -o $@ $< -lm

clean:
	rm -rf build $(LIB) oracle/liboracle.so inputs/libgen.so

.PHONY: all clean
