# Build every native artefact in-tree (the .so files travel to the GPU box with
# the gpurun snapshot; they are git-ignored).
#   libhmat.so      the product: C-ABI + sm_100a kernels (paper_2008_12441_b200/csrc)
#   liboracle.so    the CPU oracle (test infrastructure, oracle/)
#   libhgen.so      seeded input generator, host side (gen/)
#   libhgen_dev.so  seeded input generator, device side (gen/)
CUDA_HOME ?= /usr/local/cuda
NVCC      := $(CUDA_HOME)/bin/nvcc
PYSITE    := $(shell python -c 'import site,sys; print(site.getsitepackages()[0])' 2>/dev/null)
NCCL_INC  ?= $(PYSITE)/nvidia/nccl/include
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall \
             --expt-relaxed-constexpr -Xptxas -v
PKG       := paper_2008_12441_b200
CSRC      := $(PKG)/csrc

HMAT_SRC  := $(CSRC)/hmat.cpp $(CSRC)/plan.cpp $(CSRC)/comm.cpp $(CSRC)/std_exchange.cpp \
             $(CSRC)/kernels_project.cu $(CSRC)/kernels_expand.cu $(CSRC)/kernels_dmma.cu $(CSRC)/kernels_aux.cu
HMAT_HDR  := include/hmat.h $(CSRC)/plan.h $(CSRC)/kernels.h $(CSRC)/comm.h $(CSRC)/device_utils.cuh $(CSRC)/std_exchange.h $(CSRC)/geometry.cuh $(CSRC)/peer.cuh

all: $(PKG)/libhmat.so oracle/liboracle.so gen/libhgen.so gen/libhgen_dev.so

# one object per translation unit (build/obj, git-ignored), so `make -j` compiles
# the kernel files in parallel; ptxas -v output in build/obj/<file>.log
OBJDIR    := build/obj
HMAT_OBJ  := $(patsubst $(CSRC)/%,$(OBJDIR)/%.o,$(HMAT_SRC))

$(OBJDIR)/%.o: $(CSRC)/% $(HMAT_HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -Iinclude -I$(NCCL_INC) -c $< -o $@ 2> $@.log || (cat $@.log; false)

$(PKG)/libhmat.so: $(HMAT_OBJ)
	$(NVCC) $(ARCH) -shared $(HMAT_OBJ) -o $@ -ldl

oracle/liboracle.so: oracle/hmat_oracle.c gen/hgen.h
	gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared -Wall $< -o $@ -lm

gen/libhgen.so: gen/hgen_host.c gen/hgen.h
	gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared -Wall $< -o $@ -lm

gen/libhgen_dev.so: gen/hgen_device.cu gen/hgen.h
	$(NVCC) $(ARCH) -O3 -fmad=false -std=c++17 -Xcompiler -fPIC -shared $< -o $@

clean:
	rm -rf $(PKG)/libhmat.so oracle/liboracle.so gen/libhgen.so gen/libhgen_dev.so $(OBJDIR)

.PHONY: all clean
