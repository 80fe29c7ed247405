/* Prototypes of the libsodium entry points the reference's sha256.cpp / sign.cpp call, resolved
 * at link time against PyNaCl's bundled libsodium (nacl/_sodium.abi3.so). Test infrastructure
 * for oracle/_ref only (the reference links the system libsodium, proj/src/CMakeLists.txt:1). */
#pragma once
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif
#define crypto_sign_PUBLICKEYBYTES 32U
#define crypto_sign_SECRETKEYBYTES 64U
#define crypto_sign_BYTES 64U
#define crypto_hash_sha256_BYTES 32U
int sodium_init(void);
int crypto_hash_sha256(unsigned char* out, const unsigned char* in, unsigned long long inlen);
int crypto_sign_seed_keypair(unsigned char* pk, unsigned char* sk, const unsigned char* seed);
int crypto_sign_detached(unsigned char* sig, unsigned long long* siglen_p, const unsigned char* m,
                         unsigned long long mlen, const unsigned char* sk);
int crypto_sign_verify_detached(const unsigned char* sig, const unsigned char* m, unsigned long long mlen,
                                const unsigned char* pk);
#ifdef __cplusplus
}
#endif
