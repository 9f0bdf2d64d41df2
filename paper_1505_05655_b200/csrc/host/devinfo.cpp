// devinfo.cpp -- see devinfo.hpp.  The XML format is pinned against the
// reference's to_xml by tests/test_devinfo.py (same records -> same bytes).
#include "devinfo.hpp"

#include <cuda_runtime.h>

#include <sstream>

namespace gpcx::devinfo {

namespace {

std::string escape(const std::string& s) {
  std::string out;
  for (char c : s) {
    if (c == '&') out += "&amp;";
    else if (c == '<') out += "&lt;";
    else if (c == '>') out += "&gt;";
    else out += c;
  }
  return out;
}

template <class T>
void field(std::ostringstream& o, const char* tag, const T& v) {
  o << "    <" << tag << ">" << v << "</" << tag << ">\n";
}

void field(std::ostringstream& o, const char* tag, const std::array<int, 3>& v) {
  o << "    <" << tag << ">" << v[0] << " " << v[1] << " " << v[2] << "</" << tag << ">\n";
}

}  // namespace

std::vector<DeviceInfo> probe_cuda(const std::vector<int>& devices) {
  std::vector<DeviceInfo> out;
  for (int d : devices) {
    cudaDeviceProp p{};
    if (cudaGetDeviceProperties(&p, d) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    DeviceInfo i;
    i.name = p.name;
    i.compute_capability = std::to_string(p.major) + "." + std::to_string(p.minor);
    i.warp_size = p.warpSize;
    i.total_constant_memory = p.totalConstMem;
    i.total_global_memory = p.totalGlobalMem;
    i.shared_memory_per_block = p.sharedMemPerBlock;
    int khz = 0;
    if (cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, d) != cudaSuccess) cudaGetLastError();
    i.clock_rate_khz = khz;
    i.multi_processor_count = p.multiProcessorCount;
    i.registers_per_block = p.regsPerBlock;
    i.max_threads_per_block = p.maxThreadsPerBlock;
    i.max_grid_size = {p.maxGridSize[0], p.maxGridSize[1], p.maxGridSize[2]};
    i.max_threads_dim = {p.maxThreadsDim[0], p.maxThreadsDim[1], p.maxThreadsDim[2]};
    out.push_back(std::move(i));
  }
  return out;
}

std::string to_xml(std::span<const DeviceInfo> devices) {
  std::ostringstream o;
  o << "<?xml version=\"1.0\"?>\n";
  if (devices.empty()) {
    o << "<gpgpu_server/>\n";
    return o.str();
  }
  o << "<gpgpu_server>\n";
  for (std::size_t k = 0; k < devices.size(); ++k) {
    const DeviceInfo& d = devices[k];
    o << "  <device index=\"" << k << "\">\n";
    field(o, "name", escape(d.name));
    field(o, "compute_capability", escape(d.compute_capability));
    field(o, "warp_size", d.warp_size);
    field(o, "total_constant_memory", d.total_constant_memory);
    field(o, "total_global_memory", d.total_global_memory);
    field(o, "shared_memory_per_block", d.shared_memory_per_block);
    field(o, "clock_rate_khz", d.clock_rate_khz);
    field(o, "multi_processor_count", d.multi_processor_count);
    field(o, "registers_per_block", d.registers_per_block);
    field(o, "max_threads_per_block", d.max_threads_per_block);
    field(o, "max_grid_size", d.max_grid_size);
    field(o, "max_threads_dim", d.max_threads_dim);
    o << "  </device>\n";
  }
  o << "</gpgpu_server>\n";
  return o.str();
}

}  // namespace gpcx::devinfo
