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

$(PKG)/libhmat.so: $(HMAT_SRC) $(HMAT_HDR)
	$(NVCC) $(NVFLAGS) -shared -Iinclude -I$(NCCL_INC) $(HMAT_SRC) -o $@ -ldl 2> build_hmat.log || (cat build_hmat.log; false)

oracle/liboracle.so: oracle/hmat_oracle.c gen/hgen.h
	gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared -Wall $< -o $@ -lm

gen/libhgen.so: gen/hgen_host.c gen/hgen.h
	gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared -Wall $< -o $@ -lm

gen/libhgen_dev.so: gen/hgen_device.cu gen/hgen.h
	$(NVCC) $(ARCH) -O3 -fmad=false -std=c++17 -Xcompiler -fPIC -shared $< -o $@

clean:
	rm -f $(PKG)/libhmat.so oracle/liboracle.so gen/libhgen.so gen/libhgen_dev.so build_hmat.log

.PHONY: all clean
