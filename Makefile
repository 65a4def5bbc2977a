# Builds the sm_100a library (libfsx.so, C ABI in include/fsx.h) and the CPU
# oracle (test infrastructure).  `python -c "import __graft_entry__ as g; g.build()"`
# runs the same recipe.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH = -gencode arch=compute_100a,code=sm_100a
NVFLAGS = $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v -Iinclude -Ipaper_2105_06676_b200/csrc $(EXTRA)
CSRC = paper_2105_06676_b200/csrc
LIB = paper_2105_06676_b200/libfsx.so
PIPE_O = $(CSRC)/fsx_pipe.o

all: $(LIB) oracle

$(CSRC)/fsx_kernels.o: $(CSRC)/fsx_kernels.cu $(CSRC)/fsx_kernels.h $(CSRC)/fsx_device.cuh $(CSRC)/fsx_spectral.cuh $(CSRC)/fsx_async.cuh
	$(NVCC) $(NVFLAGS) -c $< -o $@ > build_ptxas.log 2>&1 || (cat build_ptxas.log; false)

$(CSRC)/fsx_pipe.o: $(CSRC)/fsx_pipe.cu $(CSRC)/fsx_kernels.h $(CSRC)/fsx_device.cuh $(CSRC)/fsx_spectral.cuh $(CSRC)/fsx_async.cuh
	$(NVCC) $(NVFLAGS) -c $< -o $@ > build_ptxas_pipe.log 2>&1 || (cat build_ptxas_pipe.log; false)

$(CSRC)/fsx_tma.o: $(CSRC)/fsx_tma.cu $(CSRC)/fsx_kernels.h $(CSRC)/fsx_device.cuh $(CSRC)/fsx_spectral.cuh $(CSRC)/fsx_async.cuh
	$(NVCC) $(NVFLAGS) -c $< -o $@ > build_ptxas_tma.log 2>&1 || (cat build_ptxas_tma.log; false)

$(CSRC)/fsx_api.o: $(CSRC)/fsx_api.cpp $(CSRC)/fsx_kernels.h include/fsx.h
	$(NVCC) $(ARCH) -O3 -std=c++17 -Xcompiler -fPIC -Iinclude -I$(CSRC) -x cu -c $< -o $@

$(CSRC)/fsx_naive.o: $(CSRC)/fsx_naive.cu $(CSRC)/fsx_kernels.h
	$(NVCC) $(NVFLAGS) -c $< -o $@ > build_ptxas_naive.log 2>&1 || (cat build_ptxas_naive.log; false)

$(CSRC)/fsx_io.o: $(CSRC)/fsx_io.cpp include/fsx.h
	g++ -std=c++20 -O2 -fPIC -Wall -Iinclude -I/usr/local/cuda/include -c $< -o $@

$(LIB): $(CSRC)/fsx_kernels.o $(CSRC)/fsx_pipe.o $(CSRC)/fsx_tma.o $(CSRC)/fsx_naive.o $(CSRC)/fsx_api.o $(CSRC)/fsx_io.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart_static -lrt -lpthread -ldl

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -f $(CSRC)/*.o $(LIB) build_ptxas*.log
	$(MAKE) -s -C oracle clean
.PHONY: all oracle clean
