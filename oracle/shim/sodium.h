// Test-infrastructure stub. libsodium is absent in this image and is used by the
// reference only for Argon2id `encapsulate_rev` (proj/src/crypto.cpp:156-169),
// which is off the Prove path. Any call fails, so encapsulate_rev throws.
#pragma once
#include <cstddef>
#define crypto_pwhash_ALG_ARGON2ID13 2
inline int sodium_init() { return -1; }
inline int crypto_pwhash(unsigned char*, unsigned long long, const char*, unsigned long long,
                         const unsigned char*, unsigned long long, std::size_t, int) {
    return -1;
}
