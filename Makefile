# Build the sm_100a C-ABI library and the CPU oracle.
#   make -j8            # both
#   make lib / oracle
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
# EXTRA / OBJDIR / LIB: A/B builds, e.g.
#   make lib EXTRA=-DGB_SRC_DELTA=0 OBJDIR=build/ab LIB=build/ab/libgosh_b200.so
EXTRA ?=
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           -Iinclude -Ipaper_2008_12336_b200/csrc --expt-relaxed-constexpr $(EXTRA)
PKG := paper_2008_12336_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJDIR ?= build/obj
OBJ := $(patsubst $(PKG)/csrc/%.cu,$(OBJDIR)/%.o,$(SRC))
HDR := $(wildcard $(PKG)/csrc/*.cuh) include/gosh_b200.h
LIB ?= $(PKG)/libgosh_b200.so

all: lib oracle

lib: $(LIB)

$(OBJDIR)/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -cudart static

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all lib oracle clean
