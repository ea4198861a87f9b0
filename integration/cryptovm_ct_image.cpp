// See cryptovm_ct_image.hpp.  Validation and error wording follow the
// reference's plaintext image code (keyservice.cpp:355-420, 427-484) and
// resolve_branch (:123-144).
#include "cryptovm_ct_image.hpp"

#include <cstring>
#include <fstream>
#include <iterator>

#include "cryptovm/errors.hpp"
#include "cryptovm/isa.hpp"

namespace cryptovm {

namespace {
constexpr char kMagic[4] = {'C', 'E', 'M', 'U'};

void put_le(std::string& out, std::uint64_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) out.push_back(static_cast<char>((v >> (8 * i)) & 0xFF));
}
std::uint64_t get_le(const char* p, int bytes) {
  std::uint64_t v = 0;
  for (int i = 0; i < bytes; ++i) v |= std::uint64_t{static_cast<std::uint8_t>(p[i])} << (8 * i);
  return v;
}

struct Header {
  unsigned width = 0;
  std::size_t count = 0;
  std::size_t blob = 0;
};

Header read_header(std::istream& in, const std::string& path, std::size_t file_size) {
  char h[kCtHeaderSize];
  if (file_size < kCtHeaderSize || !in.read(h, kCtHeaderSize))
    throw IoError("memory file truncated: " + path);
  if (std::memcmp(h, kMagic, 4) != 0) throw IoError("bad magic in memory file: " + path);
  if (static_cast<std::uint8_t>(h[4]) != kCtImageVersion)
    throw IoError("unsupported memory file version in " + path);
  Header hd;
  hd.width = static_cast<unsigned>(get_le(h + 5, 2));
  hd.count = get_le(h + 7, 4);
  hd.blob = get_le(h + 11, 4);
  if (hd.width < 1 || hd.width > 64) throw IoError("memory file has an invalid word width");
  if (hd.blob == 0) throw IoError("memory file has an invalid blob size");
  if (file_size != kCtHeaderSize + hd.count * hd.width * hd.blob)
    throw IoError("memory file truncated: " + path);
  return hd;
}

std::size_t file_size_of(const std::string& path) {
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in) throw IoError("cannot open memory file: " + path);
  return static_cast<std::size_t>(in.tellg());
}
}  // namespace

void encrypt_ct_file(Backend& key, const std::vector<std::uint64_t>& values, unsigned width,
                     const std::string& path) {
  if (width < 1 || width > 64) throw InputError("memory word width must be in [1, 64]");
  std::string out;
  std::size_t blob = 0;
  for (std::uint64_t value : values) {
    if (width < 64 && (value >> width) != 0)
      throw InputError("value " + std::to_string(value) + " does not fit in " +
                       std::to_string(width) + " bits");
    for (unsigned i = 0; i < width; ++i) {
      const std::vector<std::uint8_t> b = key.export_bit(key.encrypt_bit((value >> i) & 1));
      if (blob == 0) blob = b.size();
      if (b.size() != blob) throw Error("export_bit returned blobs of different sizes");
      out.append(reinterpret_cast<const char*>(b.data()), b.size());
    }
  }
  if (blob == 0) {  // empty image: record the backend's blob size anyway
    blob = key.export_bit(key.constant(false)).size();
  }
  std::string header(kMagic, 4);
  header.push_back(static_cast<char>(kCtImageVersion));
  put_le(header, width, 2);
  put_le(header, values.size(), 4);
  put_le(header, blob, 4);
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw IoError("cannot write memory file: " + path);
  f.write(header.data(), static_cast<std::streamsize>(header.size()));
  f.write(out.data(), static_cast<std::streamsize>(out.size()));
  if (!f) throw IoError("failed writing memory file: " + path);
}

MemoryImage decrypt_ct_file(Backend& key, const std::string& path) {
  const std::size_t size = file_size_of(path);
  std::ifstream in(path, std::ios::binary);
  const Header hd = read_header(in, path, size);
  MemoryImage image;
  image.width = hd.width;
  std::vector<std::uint8_t> blob(hd.blob);
  for (std::size_t w = 0; w < hd.count; ++w) {
    std::vector<BitHandle> bits;
    for (unsigned i = 0; i < hd.width; ++i) {
      in.read(reinterpret_cast<char*>(blob.data()), static_cast<std::streamsize>(hd.blob));
      if (!in) throw IoError("memory file truncated: " + path);
      bits.push_back(key.import_bit(blob));
    }
    std::uint64_t value = 0;
    for (unsigned i = 0; i < hd.width; ++i)
      if (key.decrypt_bit(bits[i])) value |= std::uint64_t{1} << i;
    image.values.push_back(value);
  }
  return image;
}

CiphertextFileMemory::CiphertextFileMemory(Backend& backend, const std::string& path)
    : backend_(backend), path_(path) {
  const std::size_t size = file_size_of(path);
  std::ifstream in(path, std::ios::binary);
  const Header hd = read_header(in, path, size);
  width_ = hd.width;
  count_ = hd.count;
  blob_ = hd.blob;
}

std::streamoff CiphertextFileMemory::offset_of(std::size_t address) const {
  return static_cast<std::streamoff>(kCtHeaderSize + address * width_ * blob_);
}

Word CiphertextFileMemory::load(std::size_t address) {
  if (address >= count_) {
    throw InputError("load address " + std::to_string(address) +
                     " out of range (memory has " + std::to_string(count_) + " words)");
  }
  std::ifstream in(path_, std::ios::binary);
  if (!in) throw IoError("cannot open memory file: " + path_);
  in.seekg(offset_of(address));
  std::vector<BitHandle> bits(width_);
  std::vector<std::uint8_t> blob(blob_);
  for (unsigned i = 0; i < width_; ++i) {
    in.read(reinterpret_cast<char*>(blob.data()), static_cast<std::streamsize>(blob_));
    if (!in) throw IoError("failed reading memory file: " + path_);
    bits[i] = backend_.import_bit(blob);
  }
  return Word(std::move(bits));
}

void CiphertextFileMemory::store(std::size_t address, const Word& word) {
  if (address >= count_) {
    throw InputError("store address " + std::to_string(address) +
                     " out of range (memory has " + std::to_string(count_) + " words)");
  }
  if (word.width() != width_) throw InputError("stored word width does not match the memory");
  std::string raw;
  raw.reserve(width_ * blob_);
  for (unsigned i = 0; i < width_; ++i) {
    const std::vector<std::uint8_t> b = backend_.export_bit(word.bit(i));
    if (b.size() != blob_)
      throw InputError("export_bit blob size " + std::to_string(b.size()) +
                       " does not match the image's " + std::to_string(blob_));
    raw.append(reinterpret_cast<const char*>(b.data()), b.size());
  }
  std::fstream out(path_, std::ios::binary | std::ios::in | std::ios::out);
  if (!out) throw IoError("cannot open memory file: " + path_);
  out.seekp(offset_of(address));
  out.write(raw.data(), static_cast<std::streamsize>(raw.size()));
  if (!out) throw IoError("failed writing memory file: " + path_);
}

BranchReply resolve_branch_ct(const BranchQuery& query, Backend& key, bool user_controlled) {
  const std::size_t total = query.nzcv_payload.size();
  if (total == 0 || total % 4 != 0) {
    throw ProtocolError("cannot decrypt NZCV payload: expected 4 equal flag ciphertexts, got " +
                        std::to_string(total) + " bytes");
  }
  const std::size_t blob = total / 4;
  bool flags[4];
  for (int i = 0; i < 4; ++i) {
    std::vector<std::uint8_t> b(query.nzcv_payload.begin() + i * blob,
                                query.nzcv_payload.begin() + (i + 1) * blob);
    flags[i] = key.decrypt_bit(key.import_bit(b));
  }
  const bool taken = cond_predicate(query.cond, flags[0], flags[1], flags[2], flags[3]);
  BranchReply reply;
  if (user_controlled) {
    reply.next_pc = taken ? query.target : query.fallthrough;
  } else {
    reply.taken = taken;
  }
  return reply;
}

}  // namespace cryptovm
