# Builds the B200 library and the CPU oracle. `make` = everything available here.
NVCC    ?= /usr/local/cuda/bin/nvcc
ARCH    ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS ?= -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -Xptxas -v
PKG     := paper_2207_01016_b200
CSRC    := $(PKG)/csrc
LIB     := $(PKG)/liblpd_nystrom.so
HDRS    := $(wildcard $(CSRC)/*.cuh) include/lpd_nystrom.h

all: $(LIB) oracle integration

$(CSRC)/host_widen.o: $(CSRC)/host_widen.cpp
	g++ -O3 -fPIC -c -o $@ $<

$(LIB): $(CSRC)/lpd_nystrom.cu $(HDRS) $(CSRC)/host_widen.o
	$(NVCC) $(NVFLAGS) -shared -o $@ $< $(CSRC)/host_widen.o -lcuda 2> $(PKG)/ptxas.log || (cat $(PKG)/ptxas.log; false)
	@grep -E "registers|spill|smem" $(PKG)/ptxas.log | head -20 || true

# profiling builds of the same library (LPD_LIBRARY=... selects one): K1 phase-cycle
# probe (LPD_K1_DEBUG=16) and the ablation switches (scripts/k1_ablation.sh)
variants: $(LIB)
	$(NVCC) $(NVFLAGS) -DLPD_K1_PROBE=1 -shared -o $(PKG)/liblpd_nystrom_probe.so $(CSRC)/lpd_nystrom.cu $(CSRC)/host_widen.o -lcuda 2> /dev/null
	$(NVCC) $(NVFLAGS) -DLPD_K1_ABLATIONS=1 -shared -o $(PKG)/liblpd_nystrom_ablate.so $(CSRC)/lpd_nystrom.cu $(CSRC)/host_widen.o -lcuda 2> /dev/null

oracle:
	$(MAKE) -C oracle

# the reference's own _core with compute_G served by this library (needs /root/reference)
integration: $(LIB)
	$(MAKE) -C integration

clean:
	rm -f $(LIB) $(PKG)/liblpd_nystrom_*.so $(PKG)/ptxas.log $(CSRC)/host_widen.o
	$(MAKE) -C oracle clean
	$(MAKE) -C integration clean

.PHONY: all oracle integration clean variants
